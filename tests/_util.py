"""Shared test helpers: loaders for the checkers (oracle port, compiled
reference, CPU build of the product math) and comparison utilities.

The checkers are TEST INFRASTRUCTURE (oracle/ header); nothing here is used
by the product path."""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libeig33_ref.so")
HOSTMATH_SO = os.path.join(ROOT, "tests", "hostmath", "libhostmath.so")
P = ctypes.c_void_p
S = ctypes.c_size_t


def ctypes_double(x):
    return ctypes.c_double(x)


def ptr(x):
    return None if x is None else x.ctypes.data_as(ctypes.c_void_p)


def _ensure_built():
    # both rebuild only what is stale (make / build._stale), so an edit to the
    # oracle or to eig33_math.cuh is always what the tests load
    # the compiled reference too, where its sources exist (this container; the
    # GPU box has no /root/reference and uses the prebuilt oracle/_ref .so)
    have_ref = os.path.isdir("/root/reference/proj/src")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "all" if have_ref else "port"],
                   check=True)
    from paper_2511_00292_b200 import build
    build.build_hostmath()


_port = _ref = _hm = None


def port():
    global _port
    if _port is None:
        _ensure_built()
        _port = ctypes.CDLL(PORT_SO)
    return _port


def ref():
    """Compiled reference core, or None when it is unavailable."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = ctypes.CDLL(REF_SO)
    return _ref


def hostmath():
    global _hm
    if _hm is None:
        _ensure_built()
        _hm = ctypes.CDLL(HOSTMATH_SO)
    return _hm


def nthreads():
    return max(1, min(64, os.cpu_count() or 1))


# ---- checker calls: (n,9) float64 -> outputs ----
def checker_invariants(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    out = np.empty((n, 4))
    R = ref()
    if R is not None:
        R.ref_invariants(ptr(a), S(n), ptr(out), nthreads())
    else:
        port().orc_invariants(ptr(a), S(n), ptr(out))
    return out


def checker_eigvals(a, adv=True):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    lam = np.empty((n, 3))
    fl = np.empty(n, np.uint8) if adv else None
    R = ref()
    if R is not None:
        R.ref_eigvals(ptr(a), S(n), ptr(lam), ptr(fl), nthreads())
    else:
        port().orc_eigvals(ptr(a), S(n), None, ptr(lam), ptr(fl))
    return lam, fl


def checker_eigvalss(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    lam = np.empty((n, 3))
    st = np.empty(n, np.uint8)
    R = ref()
    if R is not None:
        R.ref_eigvalss(ptr(a), S(n), ptr(lam), ptr(st), nthreads())
    else:
        port().orc_eigvalss(ptr(a), S(n), None, ptr(lam), ptr(st))
    return lam, st


# ---- comparisons ----
def bit_equal(x, y):
    """Bitwise equality with NaN == NaN regardless of sign/payload (x86 0xfff8.. vs CUDA 0x7fff..)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    return (x.view(np.uint64) == y.view(np.uint64)) | (np.isnan(x) & np.isnan(y))


TOL_UNITS = 4.0  # north_star: |lam - lam_ref| <= 4 * 2^-52 * max|lam_ref|


def lam_error_units(lam, lam_ref):
    """Per-matrix max |lam - lam_ref| in units of 2^-52 * max_k |lam_ref,k| (finite entries);
    +inf where the non-finite class differs (NaN<->NaN, +-inf<->same inf)."""
    lam = np.asarray(lam, np.float64)
    lam_ref = np.asarray(lam_ref, np.float64)
    fin = np.isfinite(lam_ref)
    cls_ok = np.where(fin, np.isfinite(lam), (np.isnan(lam) & np.isnan(lam_ref)) | (lam == lam_ref))
    scale = np.max(np.where(fin, np.abs(lam_ref), 0.0), axis=1) * 2.0 ** -52
    with np.errstate(all="ignore"):
        d = np.max(np.where(fin, np.abs(lam - lam_ref), 0.0), axis=1)
        u = np.where(d == 0, 0.0, d / np.where(scale > 0, scale, np.inf))
        u = np.where(np.isnan(u), np.inf, u)
    u = np.where(scale == 0, np.where(d == 0, 0.0, np.inf), u)
    return np.where(cls_ok.all(axis=1), u, np.inf)


def mixed_corpus(n, seed):
    """General / grid / symmetric / scalar / near-scalar / 2^k-scaled mix (host numpy)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, 9))
    q = n // 8
    with np.errstate(all="ignore"):
        a[:q] *= np.ldexp(1.0, rng.integers(-500, 501, size=(q, 1)))
    a[q:2 * q] = np.round(a[q:2 * q] * 4) / 4
    b = a[2 * q:3 * q]
    b[:, [3, 6, 7]] = b[:, [1, 2, 5]]
    c = a[3 * q:4 * q]
    c[:] = 0
    v = rng.standard_normal(q)
    c[:, 0] = c[:, 4] = c[:, 8] = v
    e = a[4 * q:5 * q]
    e *= np.ldexp(1.0, -40) * rng.random((q, 1))
    e[:, 0] += 1
    e[:, 4] += 1
    e[:, 8] += 1
    return np.ascontiguousarray(a)


KAT_MATRICES = {
    # reference tests and SURVEY Appendix B
    "diag(-1,1,2)": [-1, 0, 0, 0, 1, 0, 0, 0, 2],
    "diag(1,2,3)": [1, 0, 0, 0, 2, 0, 0, 0, 3],
    "rotation": [0, -1, 0, 1, 0, 0, 0, 0, 1],
    "sym[[2,1,0],[1,3,-1],[0,-1,4]]": [2, 1, 0, 1, 3, -1, 0, -1, 4],
    "7.25*I": [7.25, 0, 0, 0, 7.25, 0, 0, 0, 7.25],
    "3.5*I": [3.5, 0, 0, 0, 3.5, 0, 0, 0, 3.5],
    "zero": [0.0] * 9,
}


def perf_matrix():
    """fl(U1*diag(-1,1,1+1e-14)*U1^-1): reference generate_case(D2, U1, 1e-14),
    proj/src/bench.cpp:69-75 (matmul left-to-right, inverse_adjugate)."""
    u = np.array([[1, -1, 1], [1, 1, 1], [-1, -1, 1]], dtype=np.float64)
    d = np.diag([-1.0, 1.0, 1.0 + 1e-14])
    uinv = np.array([[0.5, 0, -0.5], [-0.5, 0.5, 0], [0, 0.5, 0.5]])

    def mm(x, y):
        c = np.empty((3, 3))
        for i in range(3):
            for j in range(3):
                c[i, j] = (x[i, 0] * y[0, j] + x[i, 1] * y[1, j]) + x[i, 2] * y[2, j]
        return c

    return mm(mm(u, d), uinv).reshape(9)
