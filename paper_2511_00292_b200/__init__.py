"""Batched B200 (sm_100a) evaluation of the eig33 hot path (arXiv 2511.00292).

Python mirror of the reference's public API (reference proj/python/eig33 and
proj/bindings/module.cpp:79-99: ``eigvals``, ``eigvalss``, ``invariants``,
``triple_angle``), lifted from one matrix to a contiguous batch of the same
72-byte row-major fp64 record.  Every call goes through the C ABI of
``_eig33cuda.so`` (include/eig33_cuda.h); there is no CPU fallback -- a missing
extension or a missing GPU raises.

Inputs are float64 arrays of shape (n, 3, 3) or (n, 9):
  * torch CUDA tensors -> computed in place on that device, on the current
    torch stream (device-pointer entry points, stream-ordered);
  * numpy arrays / CPU tensors -> host-buffer entry points (pinned, chunked
    H2D / kernel / D2H pipeline), results returned as numpy arrays.

Error behaviour follows the reference bindings: malformed shapes raise
ValueError (module.cpp:16-39 ``to_mat``), ``eigvalss`` on a matrix that fails
the symmetry gate raises ValueError (module.cpp turns NotSymmetric into
ValueError), CUDA failures raise RuntimeError.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "eigvals", "eigvalss", "invariants", "triple_angle", "generate", "multi_eigvals",
    "eigvals_naive", "jacobians", "VARIANTS", "generate_case", "default_delta_grid",
    "lib", "EigResult", "eps_mach", "FLAG_ADVISORY", "FLAG_NOT_SYMMETRIC",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("EIG33_SO") or os.path.join(_HERE, "_eig33cuda.so")

eps_mach = 2.0 ** -53  # reference include/eig33/mat3.hpp:10
FLAG_ADVISORY = 0x1
FLAG_NOT_SYMMETRIC = 0x2
EIG33_OK, EIG33_ECUDA, EIG33_EINVAL, EIG33_ENOTSYM = 0, 1, 2, 3

# Every symbol include/eig33_cuda.h declares (checked by tests/test_capi.py).
C_ABI_SYMBOLS = (
    "eig33cu_version", "eig33cu_last_error", "eig33cu_invariants", "eig33cu_eigvals",
    "eig33cu_eigvalss", "eig33cu_triple_angle", "eig33_invariants_host", "eig33_eigvals_host",
    "eig33_eigvalss_host", "eig33_multi_eigvals", "eig33_multi_invariants", "eig33_multi_eigvalss",
    "eig33cu_generate",
    "eig33cu_invariants_variant", "eig33cu_eigvals_naive", "eig33cu_jacobians",
    "eig33cu_generate_case", "eig33cu_disc_naive", "eig33_invariants_variant_host",
    "eig33cu_last_notsym_index", "eig33_multi_eigvals_on",
)
VARIANTS = {"Stable": 0, "Naive": 1, "NaiveTensor": 2}  # reference AlgorithmVariant

_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree extension (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise ImportError(
            f"{_SO} is missing: build it with `python -m paper_2511_00292_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(_SO)
    P, S, I, U64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
    sig = {
        "eig33cu_version": ([], I),
        "eig33cu_last_error": ([], ctypes.c_char_p),
        "eig33cu_invariants": ([P, S, P, P], I),
        "eig33cu_eigvals": ([P, S, P, P, P, P], I),
        "eig33cu_eigvalss": ([P, S, P, P, P, P], I),
        "eig33cu_triple_angle": ([P, P, S, P, P], I),
        "eig33_invariants_host": ([P, S, P, I], I),
        "eig33_eigvals_host": ([P, S, P, P, P, I], I),
        "eig33_eigvalss_host": ([P, S, P, P, P, I], I),
        "eig33_multi_eigvals": ([P, S, P, P, P, I], I),
        "eig33_multi_invariants": ([P, S, P, I], I),
        "eig33_multi_eigvalss": ([P, S, P, P, P, I], I),
        "eig33cu_generate": ([I, U64, U64, S, P, P], I),
        "eig33cu_invariants_variant": ([P, S, I, P, P], I),
        "eig33cu_eigvals_naive": ([P, S, P, P, P], I),
        "eig33cu_jacobians": ([P, S, P, P, P, P], I),
        "eig33cu_disc_naive": ([P, P, S, P, P], I),
        "eig33_invariants_variant_host": ([P, S, I, P, I], I),
        "eig33cu_generate_case": ([I, I, ctypes.c_double, P, S, P, P], I),
        "eig33cu_last_notsym_index": ([], ctypes.c_longlong),
        "eig33_multi_eigvals_on": ([P, S, P, P, P, P, I], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc == EIG33_OK:
        return
    msg = lib().eig33cu_last_error().decode(errors="replace")
    if rc == EIG33_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == EIG33_ENOTSYM:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (status {rc})")


def _torch():
    import torch  # local: numpy-only users need not import torch

    return torch


def _is_cuda_tensor(a) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, torch.Tensor) and a.is_cuda


def _records_np(a) -> np.ndarray:
    if hasattr(a, "detach") and hasattr(a, "numpy"):
        a = a.detach().cpu().numpy()
    arr = np.asarray(a)
    if arr.dtype != np.float64:
        if not (np.issubdtype(arr.dtype, np.floating) or np.issubdtype(arr.dtype, np.integer)):
            raise ValueError("matrix entries must be real numbers")
        arr = arr.astype(np.float64)
    if arr.ndim == 2 and arr.shape == (3, 3):
        arr = arr.reshape(1, 9)
    elif arr.ndim == 3 and arr.shape[1:] == (3, 3):
        arr = arr.reshape(arr.shape[0], 9)
    elif arr.ndim == 2 and arr.shape[1] == 9:
        pass
    elif arr.ndim == 1 and arr.shape[0] == 9:
        arr = arr.reshape(1, 9)
    else:
        raise ValueError(f"expected (n,3,3) or (n,9) matrices, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


def _records_cuda(a):
    torch = _torch()
    if a.dtype != torch.float64:
        raise ValueError("CUDA input must be float64")
    if a.dim() == 3 and tuple(a.shape[1:]) == (3, 3):
        a = a.reshape(a.shape[0], 9)
    elif a.dim() == 2 and a.shape[1] == 9:
        pass
    elif a.dim() == 2 and tuple(a.shape) == (3, 3):
        a = a.reshape(1, 9)
    else:
        raise ValueError(f"expected (n,3,3) or (n,9) matrices, got shape {tuple(a.shape)}")
    return a.contiguous()


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(x.data_ptr())


def _stream(a):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)


class EigResult(tuple):
    """(lam, inv, flags) with attribute access; inv / flags may be None."""

    def __new__(cls, lam, inv=None, flags=None):
        obj = super().__new__(cls, (lam, inv, flags))
        return obj

    lam = property(lambda s: s[0])
    inv = property(lambda s: s[1])
    flags = property(lambda s: s[2])

    @property
    def non_real_advisory(self):
        f = self[2]
        return None if f is None else (f & FLAG_ADVISORY) != 0


def _eig_common(entry_dev, entry_host, what, a, want_inv, want_flags, device):
    L = lib()
    if _is_cuda_tensor(a):
        torch = _torch()
        a = _records_cuda(a)
        n = a.shape[0]
        with torch.cuda.device(a.device):
            lam = torch.empty((n, 3), dtype=torch.float64, device=a.device)
            inv = torch.empty((n, 4), dtype=torch.float64, device=a.device) if want_inv else None
            flags = torch.empty((n,), dtype=torch.uint8, device=a.device) if want_flags else None
            _check(getattr(L, entry_dev)(_ptr(a), n, _ptr(inv), _ptr(lam), _ptr(flags), _stream(a)),
                   what)
        return EigResult(lam, inv, flags)
    arr = _records_np(a)
    n = arr.shape[0]
    lam = np.empty((n, 3))
    inv = np.empty((n, 4)) if want_inv else None
    flags = np.empty((n,), np.uint8) if want_flags else None
    _check(getattr(L, entry_host)(_ptr(arr), n, _ptr(inv), _ptr(lam), _ptr(flags), int(device)), what)
    return EigResult(lam, inv, flags)


def eigvals(a, *, return_invariants=False, return_flags=False, device=0) -> EigResult:
    """Batched ``eig33::eigvals`` (reference include/eig33/eigensolver.hpp:39).

    Returns EigResult(lam (n,3) ascending, inv (n,4) {i1,j2,j3,disc} or None,
    flags (n,) uint8 with bit0 = non_real_advisory, or None)."""
    return _eig_common("eig33cu_eigvals", "eig33_eigvals_host", "eigvals", a, return_invariants,
                       return_flags, device)


def eigvalss(a, *, return_invariants=False, return_flags=False, device=0) -> EigResult:
    """Batched ``eig33::eigvalss`` (reference include/eig33/eigensolver.hpp:45).

    Host inputs: raises ValueError if any matrix fails the symmetry gate, like
    the reference binding.  CUDA inputs are stream-ordered, so failures are
    reported per matrix in flags bit1 (and NaN outputs) instead of raising."""
    return _eig_common("eig33cu_eigvalss", "eig33_eigvalss_host", "eigvalss", a,
                       return_invariants, return_flags, device)


def _to_cuda(a, device):
    """Host input -> (CUDA (n,9) tensor, True) for the device-only study kernels."""
    torch = _torch()
    if _is_cuda_tensor(a):
        return _records_cuda(a), False
    return torch.from_numpy(_records_np(a)).to(f"cuda:{int(device)}"), True


def invariants(a, *, variant="Stable", device=0):
    """Batched ``eig33::invariants(a, variant)`` (reference invariants.hpp:74):
    (n,4) {i1,j2,j3,disc}; variant "Stable" (the hot path), "Naive" or "NaiveTensor"."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown AlgorithmVariant {variant!r}")
    if variant != "Stable":
        if _is_cuda_tensor(a):
            torch = _torch()
            d = _records_cuda(a)
            with torch.cuda.device(d.device):
                out = torch.empty((d.shape[0], 4), dtype=torch.float64, device=d.device)
                _check(lib().eig33cu_invariants_variant(_ptr(d), d.shape[0], VARIANTS[variant],
                                                        _ptr(out), _stream(d)), "invariants")
            return out
        arr = _records_np(a)
        out = np.empty((arr.shape[0], 4))
        _check(lib().eig33_invariants_variant_host(_ptr(arr), arr.shape[0], VARIANTS[variant], _ptr(out),
                                                   int(device)), "invariants")
        return out
    L = lib()
    if _is_cuda_tensor(a):
        torch = _torch()
        a = _records_cuda(a)
        with torch.cuda.device(a.device):
            inv = torch.empty((a.shape[0], 4), dtype=torch.float64, device=a.device)
            _check(L.eig33cu_invariants(_ptr(a), a.shape[0], _ptr(inv), _stream(a)), "invariants")
        return inv
    arr = _records_np(a)
    inv = np.empty((arr.shape[0], 4))
    _check(L.eig33_invariants_host(_ptr(arr), arr.shape[0], _ptr(inv), int(device)), "invariants")
    return inv


def eigvals_naive(a, *, return_flags=False, device=0) -> EigResult:
    """Batched ``eig33::eigvals_naive`` (reference eigensolver.hpp:49): the
    error-study path fed by the naive invariants."""
    torch = _torch()
    d, host = _to_cuda(a, device)
    with torch.cuda.device(d.device):
        lam = torch.empty((d.shape[0], 3), dtype=torch.float64, device=d.device)
        fl = torch.empty((d.shape[0],), dtype=torch.uint8, device=d.device) if return_flags else None
        _check(lib().eig33cu_eigvals_naive(_ptr(d), d.shape[0], _ptr(lam), _ptr(fl), _stream(d)),
               "eigvals_naive")
    if host:
        return EigResult(lam.cpu().numpy(), None, None if fl is None else fl.cpu().numpy())
    return EigResult(lam, None, fl)


def jacobians(a, *, device=0):
    """Batched ``eig33::jacobian_j2 / jacobian_j3 / jacobian_disc`` (reference
    invariants.hpp:62-69): three (n,3,3) row-major gradients."""
    torch = _torch()
    d, host = _to_cuda(a, device)
    n = d.shape[0]
    with torch.cuda.device(d.device):
        outs = [torch.empty((n, 9), dtype=torch.float64, device=d.device) for _ in range(3)]
        _check(lib().eig33cu_jacobians(_ptr(d), n, *(_ptr(o) for o in outs), _stream(d)), "jacobians")
    outs = [o.view(n, 3, 3) for o in outs]
    return tuple(o.cpu().numpy() for o in outs) if host else tuple(outs)


def _vec_cuda(x, device):
    """1-D float64 CUDA view of x; host input is copied to cuda:device (then
    the result goes back to the host as numpy)."""
    torch = _torch()
    if _is_cuda_tensor(x):
        if x.dtype != torch.float64:
            raise ValueError("CUDA input must be float64")
        return x.reshape(-1).contiguous(), False
    arr = np.asarray(x)
    if not (np.issubdtype(arr.dtype, np.floating) or np.issubdtype(arr.dtype, np.integer)):
        raise ValueError("entries must be real numbers")
    arr = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1)
    return torch.from_numpy(arr).to(f"cuda:{int(device)}"), True


def _pairwise(entry, what, x, y, device):
    torch = _torch()
    xd, host = _vec_cuda(x, device)
    yd, _ = _vec_cuda(y, xd.device.index)
    if xd.shape != yd.shape:
        raise ValueError(f"{what}: arguments must have equal length")
    out = torch.empty_like(xd)
    with torch.cuda.device(xd.device):
        _check(getattr(lib(), entry)(_ptr(xd), _ptr(yd), xd.numel(), _ptr(out), _stream(xd)), what)
    return out.cpu().numpy() if host else out


def triple_angle(j3, disc, *, device=0):
    """Batched ``eig33::triple_angle`` (eigensolver.hpp:21): phi for each
    (j3, disc) pair; CUDA float64 tensors in -> tensor out, host arrays -> numpy."""
    return _pairwise("eig33cu_triple_angle", "triple_angle", j3, disc, device)


def disc_naive(j2, j3, *, device=0):
    """Batched ``eig33::disc_naive(j2, j3)`` (invariants.hpp:59, src/invariants.cpp:58):
    ((4 j2) j2) j2 - (27 j3) j3 for each pair, on the GPU."""
    return _pairwise("eig33cu_disc_naive", "disc_naive", j2, j3, device)


def generate(config: int, n: int, seed: int = 0, first_index: int = 0, device="cuda"):
    """Synthetic corpus of BASELINE config 1..5 as an (n,9) CUDA float64 tensor."""
    torch = _torch()
    out = torch.empty((n, 9), dtype=torch.float64, device=device)
    with torch.cuda.device(out.device):
        _check(lib().eig33cu_generate(int(config), int(seed) & (2**64 - 1), int(first_index), int(n),
                                      _ptr(out), _stream(out)), "generate")
    return out


PATHS = {"D1": 0, "D2": 1}                    # reference PathKind (bench.hpp:21)
TRANSFORMS = {"Symm": 0, "U1": 1, "U2": 2}    # reference Transform::Kind (bench.hpp:28-31)


def default_delta_grid():
    """The reference's sweep grid 10^(-k/4), k = 4..64 (src/bench.cpp:77-82)."""
    return [10.0 ** (-k / 4.0) for k in range(4, 65)]


def generate_case(path: str, transform: str, deltas, gamma: float = 1e-3, device="cuda"):
    """Batched ``eig33::bench::generate_case`` (reference src/bench.cpp:53-75):
    one (n,9) CUDA record per delta, bit-identical to the reference."""
    torch = _torch()
    if path not in PATHS or transform not in TRANSFORMS:
        raise ValueError("path must be D1/D2 and transform Symm/U1/U2")
    d = torch.as_tensor(np.asarray(deltas, dtype=np.float64).reshape(-1), device=device)
    out = torch.empty((d.numel(), 9), dtype=torch.float64, device=device)
    with torch.cuda.device(out.device):
        _check(lib().eig33cu_generate_case(PATHS[path], TRANSFORMS[transform], float(gamma), _ptr(d),
                                           d.numel(), _ptr(out), _stream(out)), "generate_case")
    return out


def multi_eigvals(a, ngpu: int = None, *, devices=None, return_invariants=False,
                  return_flags=False) -> EigResult:
    """Host batch sharded over devices 0..ngpu-1 (eig33_multi_eigvals), or over
    an explicit per-shard device list (eig33_multi_eigvals_on)."""
    arr = _records_np(a)
    n = arr.shape[0]
    lam = np.empty((n, 3))
    inv = np.empty((n, 4)) if return_invariants else None
    flags = np.empty((n,), np.uint8) if return_flags else None
    if devices is not None:
        d = np.ascontiguousarray(np.asarray(devices, dtype=np.int32).reshape(-1))
        _check(lib().eig33_multi_eigvals_on(_ptr(arr), n, _ptr(inv), _ptr(lam), _ptr(flags), _ptr(d),
                                            int(d.size)), "multi_eigvals")
    else:
        _check(lib().eig33_multi_eigvals(_ptr(arr), n, _ptr(inv), _ptr(lam), _ptr(flags), int(ngpu)),
               "multi_eigvals")
    return EigResult(lam, inv, flags)


def multi_eigvalss(a, ngpu: int, *, return_invariants=False, return_flags=False) -> EigResult:
    """Host batch sharded over devices 0..ngpu-1 (eig33_multi_eigvalss);
    ValueError if any matrix fails the symmetry gate."""
    arr = _records_np(a)
    n = arr.shape[0]
    lam = np.empty((n, 3))
    inv = np.empty((n, 4)) if return_invariants else None
    flags = np.empty((n,), np.uint8) if return_flags else None
    _check(lib().eig33_multi_eigvalss(_ptr(arr), n, _ptr(inv), _ptr(lam), _ptr(flags), int(ngpu)),
           "multi_eigvalss")
    return EigResult(lam, inv, flags)


def multi_invariants(a, ngpu: int) -> np.ndarray:
    """Host batch sharded over devices 0..ngpu-1 (eig33_multi_invariants): (n,4)."""
    arr = _records_np(a)
    inv = np.empty((arr.shape[0], 4))
    _check(lib().eig33_multi_invariants(_ptr(arr), arr.shape[0], _ptr(inv), int(ngpu)), "multi_invariants")
    return inv
