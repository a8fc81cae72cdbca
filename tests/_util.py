"""Shared test helpers: loaders for the checkers (compiled reference core --
the parity checker, hard-required --, oracle port, CPU build of the product
math, host corpus regeneration) and comparison utilities.

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
    """The compiled reference core (oracle/_ref).  There is no fallback: every
    parity check runs against the reference's own code, so a missing build is
    an error, never a silent switch to the port."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference "
                                    "exists (the prebuilt .so travels to the GPU box)")
        _ref = ctypes.CDLL(REF_SO)
    return _ref


CHECKER = "compiled reference core (oracle/_ref/libeig33_ref.so)"


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
    ref().ref_invariants(ptr(a), S(n), ptr(out), nthreads())
    return out


def checker_eigvals(a, adv=True):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    lam = np.empty((n, 3))
    fl = np.empty(n, np.uint8) if adv else None
    ref().ref_eigvals(ptr(a), S(n), ptr(lam), ptr(fl), nthreads())
    return lam, fl


def checker_eigvalss(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    lam = np.empty((n, 3))
    st = np.empty(n, np.uint8)
    ref().ref_eigvalss(ptr(a), S(n), ptr(lam), ptr(st), nthreads())
    return lam, st


# ---- comparisons ----
def bit_equal(x, y):
    """Bitwise equality with NaN == NaN regardless of sign/payload (x86 0xfff8.. vs CUDA 0x7fff..)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    return (x.view(np.uint64) == y.view(np.uint64)) | (np.isnan(x) & np.isnan(y))


TOL_UNITS = 4.0  # north_star: |lam - lam_ref| <= 4 ulp * max|lam_ref|, both readings below


def lam_error_ulps(lam, lam_ref):
    """Strict reading of the north_star gate: per-matrix max |lam - lam_ref| in
    units of ulp(max_k |lam_ref,k|) (np.spacing: the binade's ulp, 2^(e-52) for
    max|lam_ref| in [2^e, 2^(e+1))).  Up to 2x tighter than lam_error_units;
    +inf where the non-finite class differs."""
    lam = np.asarray(lam, np.float64)
    lam_ref = np.asarray(lam_ref, np.float64)
    fin = np.isfinite(lam_ref)
    cls_ok = np.where(fin, np.isfinite(lam), (np.isnan(lam) & np.isnan(lam_ref)) | (lam == lam_ref))
    mx = np.max(np.where(fin, np.abs(lam_ref), 0.0), axis=1)
    ulp = np.spacing(mx)  # spacing(0) = 2^-1074, the smallest ulp
    with np.errstate(all="ignore"):
        d = np.max(np.where(fin, np.abs(lam - lam_ref), 0.0), axis=1)
        u = np.where(d == 0, 0.0, d / ulp)
        u = np.where(np.isnan(u), np.inf, u)
    return np.where(cls_ok.all(axis=1), u, np.inf)


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


CORPUS_SO = os.path.join(ROOT, "oracle", "libcorpus.so")
_corpus = None


def host_corpus(config, n, seed, first=0, threads=None):
    """Records [first, first+n) of BASELINE config 1..5 regenerated on the host
    (oracle/corpus_host.cpp over the shared recipes eig33_gen_core.h):
    bit-identical to the device generator eig33cu_generate."""
    global _corpus
    if _corpus is None:
        _ensure_built()
        _corpus = ctypes.CDLL(CORPUS_SO)
        _corpus.corpus_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, S, P,
                                            ctypes.c_int]
    a = np.empty((n, 9))
    rc = _corpus.corpus_generate(config, seed & (2 ** 64 - 1), first, n, ptr(a), threads or nthreads())
    assert rc == 0
    return a


_libm = None


def _glibc():
    global _libm
    if _libm is None:
        _libm = ctypes.CDLL("libm.so.6")
        for f in ("atan2",):
            getattr(_libm, f).restype = ctypes.c_double
            getattr(_libm, f).argtypes = [ctypes.c_double, ctypes.c_double]
        for f in ("sin", "cos"):
            getattr(_libm, f).restype = ctypes.c_double
            getattr(_libm, f).argtypes = [ctypes.c_double]
    return _libm


def libm_misrounds(inv_row):
    """Does this host's libm -- the atan2 / sincos the reference calls at
    proj/src/eigensolver.cpp:88 and :21 -- return a not-correctly-rounded
    result for the transcendental arguments of this record (invariants
    inv_row)?  Returns the names of the misrounded calls (mpmath at 200 bits
    decides the correctly rounded value)."""
    import math

    import mpmath

    i1, j2, j3, disc = (float(x) for x in inv_row)
    if not (j2 > 0.0) or not math.isfinite(j3) or not math.isfinite(disc):
        return []
    M = _glibc()
    y = math.sqrt(27.0 * (disc if disc > 0.0 else 0.0))
    x = 27.0 * j3
    bad = []
    with mpmath.workprec(200):
        phi = M.atan2(y, x)
        if phi != float(mpmath.atan2(mpmath.mpf(y), mpmath.mpf(x))):
            bad.append("atan2")
        th = phi / 3.0
        if M.sin(th) != float(mpmath.sin(mpmath.mpf(th))):
            bad.append("sin")
        if M.cos(th) != float(mpmath.cos(mpmath.mpf(th))):
            bad.append("cos")
    return bad


STRICT_UNITS = 4.0  # north_star, strict reading: 4 * ulp(max|lam_ref|)


def lam_gate(a, lam, lam_ref, inv_ref=None, fallback=None):
    """The eigenvalue gate, strict reading: every record within
    4 * ulp(max|lam_ref|) of the reference, except records where the
    reference's libm misrounded one of its transcendental calls for that very
    record (the device path is correctly rounded there, so the two cannot
    agree to the last bit) -- those must still be inside the loose reading
    4 * 2^-52 * max|lam_ref| -- or records `fallback(a, lam, lam_ref)` accepts
    (config 4: the north_star's forward-error criterion).  Returns (strict
    errors, loose errors, indices of the explained exceptions); raises
    AssertionError with the first offenders otherwise."""
    es = lam_error_ulps(lam, lam_ref)
    el = lam_error_units(lam, lam_ref)
    over = np.nonzero(es > STRICT_UNITS)[0]
    if over.size and fallback is not None:
        ok = fallback(a[over], lam[over], lam_ref[over])
        over = over[~ok]
    explained = []
    if over.size:
        assert over.size <= 1000, f"{over.size} records over {STRICT_UNITS} ulp(max|lam|)"
        if inv_ref is None:
            inv_ref = checker_invariants(a[over])
            rows = inv_ref
        else:
            rows = inv_ref[over]
        bad = []
        for k, i in enumerate(over):
            if el[i] <= TOL_UNITS and libm_misrounds(rows[k]):
                explained.append(int(i))
            else:
                bad.append(int(i))
        assert not bad, (f"{len(bad)} records over {STRICT_UNITS} ulp(max|lam_ref|) without a libm "
                         f"misrounding behind them: first {bad[:5]}, strict {es[bad[:5]]}, loose {el[bad[:5]]}")
    return es, el, explained


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
