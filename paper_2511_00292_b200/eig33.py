"""Drop-in for the reference's Python module (``import eig33``: the pybind11
extension ``_eig33``, reference bindings/module.cpp:53-108 re-exported by
python/eig33/__init__.py).

Same names, argument forms, return types and errors, computed by this
package's sm_100a kernels:

* a single matrix -- 9 flat numbers or 3 rows of 3 (``to_mat``,
  bindings/module.cpp:16-39), or a (3,3) / (9,) array -- returns what the
  reference returns: ``EigenTriple`` for the eigenvalue solvers, ``float`` for
  the invariants, a list of 3 row lists for the Jacobians;
* a batch -- an (n,3,3) or (n,9) numpy array or CUDA float64 tensor -- returns
  arrays (numpy for host input, tensors for CUDA input): the batched surface
  the reference module does not have.

Errors follow the reference binding: malformed matrices and asymmetric input
to ``eigvalss`` raise ``ValueError``.  There is no CPU path: without the CUDA
library every call raises.
"""
from collections.abc import Sequence

import numpy as np

from . import (FLAG_ADVISORY, EigResult, _is_cuda_tensor, _records_cuda, _records_np)
from . import disc_naive as _disc_naive_batch
from . import eigvals as _eigvals
from . import eigvals_naive as _eigvals_naive
from . import eigvalss as _eigvalss
from . import invariants as _invariants
from . import jacobians as _jacobians

__all__ = ["EigenTriple", "eps_mach", "eigvals", "eigvalss", "eigvals_naive", "i1", "j2_stable",
           "j2_naive", "j2_tensor", "j3_stable", "j3_naive", "j3_tensor", "disc_stable",
           "disc_naive", "jacobian_j2", "jacobian_j3", "jacobian_disc"]

eps_mach = 2.0 ** -53  # include/eig33/mat3.hpp:10


class EigenTriple:
    """``eig33::EigenTriple`` as the reference binding exposes it
    (bindings/module.cpp:57-75): lambda1 <= lambda2 <= lambda3, non_real_advisory,
    len() == 3, indexing, the same repr."""

    __slots__ = ("lambda1", "lambda2", "lambda3", "non_real_advisory")

    def __init__(self, l1, l2, l3, adv=False):
        self.lambda1, self.lambda2, self.lambda3 = float(l1), float(l2), float(l3)
        self.non_real_advisory = bool(adv)

    def __len__(self):
        return 3

    def __getitem__(self, i):
        i = int(i)
        i = i + 3 if i < 0 else i
        if i == 0:
            return self.lambda1
        if i == 1:
            return self.lambda2
        if i == 2:
            return self.lambda3
        raise IndexError("EigenTriple index out of range")

    def __repr__(self):
        return (f"EigenTriple({self.lambda1!r}, {self.lambda2!r}, {self.lambda3!r}"
                + (", non_real_advisory=True)" if self.non_real_advisory else ")"))


def _to_mat(obj) -> np.ndarray:
    """bindings/module.cpp:16-39: 9 flat entries (row-major) or 3 rows of 3."""
    if not isinstance(obj, Sequence) or isinstance(obj, (str, bytes)):
        raise ValueError("matrix must be a sequence of numbers")
    n = len(obj)
    try:
        if n == 9:
            return np.array([float(x) for x in obj], dtype=np.float64).reshape(1, 9)
        if n == 3:
            rows = []
            for row in obj:
                if not isinstance(row, Sequence) or isinstance(row, (str, bytes)):
                    raise ValueError("matrix must be 9 flat entries or 3 rows of 3")
                if len(row) != 3:
                    raise ValueError("rows must have 3 entries")
                rows.extend(float(x) for x in row)
            return np.array(rows, dtype=np.float64).reshape(1, 9)
    except TypeError as e:  # a non-numeric entry
        raise ValueError(f"matrix entries must be numbers ({e})") from None
    raise ValueError("matrix must be 9 flat entries or 3 rows of 3")


def _parse(a):
    """(records, single): records is an (n,9) float64 numpy array or CUDA tensor."""
    if _is_cuda_tensor(a):
        single = tuple(a.shape) in ((3, 3), (9,))
        return _records_cuda(a.reshape(1, 9) if single else a), single
    if isinstance(a, np.ndarray):
        single = a.shape in ((3, 3), (9,))
        return _records_np(a.reshape(1, 9) if single else a), single
    return _to_mat(a), True


def _host(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else x


def _triple(r: EigResult) -> EigenTriple:
    lam, flags = _host(r.lam), _host(r.flags)
    return EigenTriple(lam[0, 0], lam[0, 1], lam[0, 2], bool(flags[0] & FLAG_ADVISORY))


def eigvals(a):
    """Ascending eigenvalues by the stable closed-form solver (``eig33::eigvals``)."""
    recs, single = _parse(a)
    r = _eigvals(recs, return_flags=True)
    return _triple(r) if single else r


def eigvalss(a):
    """Ascending eigenvalues for symmetric input; ValueError otherwise (``eig33::eigvalss``).
    A CUDA batch reports rejects in flags bit 1 instead (stream-ordered)."""
    recs, single = _parse(a)
    if single and _is_cuda_tensor(recs):
        recs = recs.cpu().numpy()  # one matrix: raise like the reference
    r = _eigvalss(recs, return_flags=True)
    if single:
        return EigenTriple(*_host(r.lam)[0], False)
    return r


def eigvals_naive(a):
    """Ascending eigenvalues from the textbook invariant formulas (``eig33::eigvals_naive``)."""
    recs, single = _parse(a)
    r = _eigvals_naive(recs, return_flags=True)
    return _triple(r) if single else r


def _inv(a, variant, col):
    recs, single = _parse(a)
    v = _invariants(recs, variant=variant)[:, col]
    return float(_host(v)[0]) if single else v


def i1(a):
    """First invariant (trace), ``eig33::i1``."""
    return _inv(a, "Stable", 0)


def j2_stable(a):
    """J2 by the paper's stable formula, ``eig33::j2_stable``."""
    return _inv(a, "Stable", 1)


def j3_stable(a):
    """J3 by the stable formula, ``eig33::j3_stable``."""
    return _inv(a, "Stable", 2)


def disc_stable(a):
    """Discriminant by the stable sum of products, ``eig33::disc_stable``."""
    return _inv(a, "Stable", 3)


def j2_naive(a):
    """J2 from I1 and I2 (``eig33::j2_naive``)."""
    return _inv(a, "Naive", 1)


def j3_naive(a):
    """J3 from I1, I2, I3 (``eig33::j3_naive``)."""
    return _inv(a, "Naive", 2)


def j2_tensor(a):
    """J2 = tr(s^2)/2 of the deviator (``eig33::j2_tensor``)."""
    return _inv(a, "NaiveTensor", 1)


def j3_tensor(a):
    """J3 = det(s) of the deviator (``eig33::j3_tensor``)."""
    return _inv(a, "NaiveTensor", 2)


def disc_naive(j2, j3):
    """4 j2^3 - 27 j3^2 in the reference's order (``eig33::disc_naive``);
    scalars give a float, arrays an array."""
    if np.ndim(j2) == 0 and np.ndim(j3) == 0 and not _is_cuda_tensor(j2):
        return float(_disc_naive_batch(np.array([float(j2)]), np.array([float(j3)]))[0])
    return _disc_naive_batch(j2, j3)


def _jac(a, k):
    recs, single = _parse(a)
    g = _jacobians(recs)[k]
    if single:
        return [[float(x) for x in row] for row in _host(g)[0]]
    return g


def jacobian_j2(a):
    """dJ2/dA (``eig33::jacobian_j2``): rows of 3."""
    return _jac(a, 0)


def jacobian_j3(a):
    """dJ3/dA (``eig33::jacobian_j3``): rows of 3."""
    return _jac(a, 1)


def jacobian_disc(a):
    """d disc/dA (``eig33::jacobian_disc``): rows of 3."""
    return _jac(a, 2)
