"""Generate tests/golden/eig33_golden.npz from the COMPILED REFERENCE
(oracle/_ref/libeig33_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Corpus (seeded, numpy): the reference tests' known-answer matrices, the perf
matrix, scaled identities (test_eigensolver.cpp:41-52, acceptance C2),
symmetric matrices, and a small mixed corpus with 2^k scaling, grids,
near-scalar and non-finite-producing entries.  Stored: inputs, invariants
(bitwise), eigvals lambda + advisory, eigvalss lambda + NotSymmetric status,
triple_angle KATs.  lambda bits depend on this host's libm (glibc 2.39, x86-64);
tests compare them within the 4-ulp tolerance, invariants and flags bitwise."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests import _util as U  # noqa: E402


def corpus():
    rng = np.random.default_rng(20251100)
    rows = [np.array(v, dtype=np.float64) for v in U.KAT_MATRICES.values()]
    rows.append(U.perf_matrix())
    alphas = np.ldexp(rng.uniform(-1, 1, 64), rng.integers(-30, 31, 64))
    alphas = np.concatenate([alphas, 10.0 ** rng.uniform(-100, 100, 64)])
    for al in alphas:
        rows.append(np.array([al, 0, 0, 0, al, 0, 0, 0, al]))
    sym = rng.uniform(-5, 5, (256, 9))
    sym[:, [3, 6, 7]] = sym[:, [1, 2, 5]]
    rows.extend(sym)
    mixed = U.mixed_corpus(1536, 7)
    rows.extend(mixed)
    extremes = np.array([[1e200, 2e200, -1e200, 3e199, 1e200, 0, 0, 5e199, -2e200],
                         [1e-200, 2e-200, 0, -1e-200, 3e-200, 1e-200, 0, 0, 2e-200],
                         [np.inf, 0, 0, 0, 1, 0, 0, 0, 2],
                         [np.nan, 0, 0, 0, 1, 0, 0, 0, 2],
                         [1, 1e-300, 0, 1e-300, 1, 0, 0, 0, 1]])
    rows.extend(extremes)
    return np.ascontiguousarray(np.array(rows, dtype=np.float64))


def main():
    R = U.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libeig33_ref.so missing: run `make -C oracle ref` first")
    a = corpus()
    n = a.shape[0]
    inv = np.empty((n, 4))
    R.ref_invariants(U.ptr(a), U.S(n), U.ptr(inv), 1)
    lam = np.empty((n, 3))
    adv = np.empty(n, np.uint8)
    R.ref_eigvals(U.ptr(a), U.S(n), U.ptr(lam), U.ptr(adv), 1)
    slam = np.empty((n, 3))
    sst = np.empty(n, np.uint8)
    R.ref_eigvalss(U.ptr(a), U.S(n), U.ptr(slam), U.ptr(sst), 1)
    ta_in = np.array([[0.0, 27.0], [5.0, 0.0], [-5.0, 0.0], [1.0, -5.0], [-0.0, 0.0], [0.0, 0.0],
                      [np.inf, 1.0], [-np.inf, 1.0], [1.0, np.inf], [np.nan, 1.0], [1.0, np.nan],
                      [-20.0 / 27.0, 36.0], [1e-300, 1e-300], [3.0, 1e300], [-1e300, 4.0]])
    ta = np.empty(len(ta_in))
    j3 = np.ascontiguousarray(ta_in[:, 0])
    dc = np.ascontiguousarray(ta_in[:, 1])
    R.ref_triple_angle(U.ptr(j3), U.ptr(dc), U.S(len(ta_in)), U.ptr(ta))
    out = os.path.join(HERE, "eig33_golden.npz")
    np.savez_compressed(out, a=a, inv=inv, lam=lam, adv=adv, sym_lam=slam, sym_status=sst,
                        ta_in=ta_in, ta=ta)
    print("wrote", out, n, "records")


if __name__ == "__main__":
    main()
