"""Pin the checkers before trusting them (CPU only).

* the C restatement (oracle/eig33_oracle.c) against the compiled reference
  core (oracle/_ref) bitwise on mixed corpora, including the advisory flag and
  eigvalss' NotSymmetric status;
* both against the committed golden fixtures (made by the compiled reference,
  tests/golden/make_golden.py);
* the known answers asserted by the reference's own tests
  (proj/tests/test_invariants.cpp, test_eigensolver.cpp, python/test_smoke.py,
  acceptance.cpp C1/C2) and SURVEY Appendix B bit patterns.
"""
import math
import os

import numpy as np
import pytest

from tests import _util as U

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "eig33_golden.npz")


def _port_inv(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    out = np.empty((a.shape[0], 4))
    U.port().orc_invariants(U.ptr(a), U.S(a.shape[0]), U.ptr(out))
    return out


def _port_eig(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    lam = np.empty((n, 3))
    adv = np.empty(n, np.uint8)
    U.port().orc_eigvals(U.ptr(a), U.S(n), None, U.ptr(lam), U.ptr(adv))
    return lam, adv


def _port_sym(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 9)
    n = a.shape[0]
    lam = np.empty((n, 3))
    st = np.empty(n, np.uint8)
    U.port().orc_eigvalss(U.ptr(a), U.S(n), None, U.ptr(lam), U.ptr(st))
    return lam, st


def _bits(x):
    return np.float64(x).view(np.uint64).item()


def test_port_matches_golden_fixtures():
    g = np.load(GOLDEN)
    inv = _port_inv(g["a"])
    assert U.bit_equal(inv, g["inv"]).all()
    lam, adv = _port_eig(g["a"])
    assert (adv == g["adv"]).all()
    assert (U.lam_error_units(lam, g["lam"]) <= U.TOL_UNITS).all()
    slam, sst = _port_sym(g["a"])
    assert (sst == g["sym_status"]).all()
    ok = sst == 0
    assert (U.lam_error_units(slam[ok], g["sym_lam"][ok]) <= U.TOL_UNITS).all()


def test_port_bitwise_equals_compiled_reference():
    a = U.mixed_corpus(1 << 17, 3)
    inv_r = np.empty((a.shape[0], 4))
    U.ref().ref_invariants(U.ptr(a), U.S(a.shape[0]), U.ptr(inv_r), U.nthreads())
    assert U.bit_equal(_port_inv(a), inv_r).all()
    lam_r, adv_r = U.checker_eigvals(a)
    lam, adv = _port_eig(a)
    assert U.bit_equal(lam, lam_r).all()  # same host libm -> same bits
    assert (adv == adv_r).all()
    slam_r, sst_r = U.checker_eigvalss(a)
    slam, sst = _port_sym(a)
    assert (sst == sst_r).all()
    assert U.bit_equal(slam, slam_r).all()


def test_kat_invariants():
    inv = _port_inv(np.array(U.KAT_MATRICES["diag(-1,1,2)"]))[0]
    # acceptance C1 (acceptance.cpp:50-60), python smoke :49-55, Appendix B bits
    assert inv[0] == 2.0 and inv[3] == 36.0
    assert _bits(inv[1]) == 0x4002AAAAAAAAAAAB and _bits(inv[2]) == 0xBFE7B425ED097B42
    inv = _port_inv(np.array(U.KAT_MATRICES["diag(1,2,3)"]))[0]
    assert inv[1] == 1.0 and inv[2] == 0.0 and inv[3] == 4.0  # test_invariants.cpp:61,124
    inv = _port_inv(np.array(U.KAT_MATRICES["rotation"]))[0]
    assert inv[3] == -16.0  # test_eigensolver.cpp:71-81
    inv = _port_inv(np.array(U.KAT_MATRICES["3.5*I"]))[0]
    assert inv[3] == 0.0  # test_invariants.cpp:158
    inv = _port_inv(U.perf_matrix())[0]  # Appendix B perf matrix
    assert [_bits(x) for x in inv] == [0x3FF000000000002C, 0x3FF5555555555573, 0xBFE2F684BDA12F8F,
                                       0x3A5F620000000030]
    u1 = np.array([[1, -1, 1], [1, 1, 1], [-1, -1, 1]], dtype=np.float64)
    u1inv = np.array([[0.5, 0, -0.5], [-0.5, 0.5, 0], [0, 0.5, 0.5]])
    a = (u1 @ np.diag([-1.0, 1, 2]) @ u1inv).reshape(9)  # exact (dyadic), test_invariants.cpp:53-56
    assert _port_inv(a)[0][0] == 2.0


def test_kat_scaled_identities_annihilate():
    rng = np.random.default_rng(31)
    al = np.concatenate([np.ldexp(rng.uniform(-1, 1, 200), rng.integers(-30, 31, 200)),
                         10.0 ** rng.uniform(-100, 100, 1000)])
    a = np.zeros((al.size, 9))
    a[:, 0] = a[:, 4] = a[:, 8] = al
    inv = _port_inv(a)
    assert (inv[:, 1:] == 0).all()
    lam, adv = _port_eig(a)
    assert (lam == al[:, None]).all() and not adv.any()  # test_eigensolver.cpp:41-52, acceptance C2


def test_kat_eigvals_and_advisory():
    lam, adv = _port_eig(np.array(U.KAT_MATRICES["rotation"]))
    assert adv[0] == 1 and np.isfinite(lam).all()
    lam, adv = _port_eig(np.array(U.KAT_MATRICES["diag(1,2,3)"]))
    assert np.abs(lam[0] - [1, 2, 3]).max() <= 1e-14 and adv[0] == 0  # cli test_cli.py:18-28
    lam, _ = _port_eig(np.array(U.KAT_MATRICES["7.25*I"]))
    assert (lam == 7.25).all()


def test_kat_triple_angle():
    P = U.port()
    P.orc_triple_angle.restype = __import__("ctypes").c_double
    P.orc_triple_angle.argtypes = [__import__("ctypes").c_double] * 2
    assert P.orc_triple_angle(0.0, 27.0) == math.pi / 2  # test_eigensolver.cpp:30-39
    assert P.orc_triple_angle(5.0, 0.0) == 0.0
    assert P.orc_triple_angle(-5.0, 0.0) == math.pi
    assert P.orc_triple_angle(1.0, -5.0) == 0.0
    assert abs(P.orc_triple_angle(-20.0 / 27.0, 36.0) - 2.141173136834297) <= 1e-14


def test_eigvalss_symmetry_gate():
    a = np.array([[1.0, 1.0, 0, 1.0 + 1e-8, 2, 0, 0, 0, 3],
                  U.KAT_MATRICES["rotation"],
                  [1.0, 1.0, 0, 1.0 + 2.0 ** -52, 2, 0, 0, 0, 3]])
    _, st = _port_sym(a)
    assert list(st) == [1, 1, 0]  # test_eigensolver.cpp:150-165


def test_port_study_variants_bitwise_equal_compiled_reference():
    """naive / tensor invariants, eigvals_naive, Jacobians."""
    a = U.mixed_corpus(1 << 15, 23)
    n = a.shape[0]
    P, R = U.port(), U.ref()
    for v in (1, 2):
        x, y = np.empty((n, 4)), np.empty((n, 4))
        P.orc_invariants_variant(U.ptr(a), U.S(n), v, U.ptr(x))
        R.ref_invariants_variant(U.ptr(a), U.S(n), v, U.ptr(y), U.nthreads())
        assert U.bit_equal(x, y).all()
    l1, l2 = np.empty((n, 3)), np.empty((n, 3))
    f1, f2 = np.empty(n, np.uint8), np.empty(n, np.uint8)
    P.orc_eigvals_naive(U.ptr(a), U.S(n), U.ptr(l1), U.ptr(f1))
    R.ref_eigvals_naive(U.ptr(a), U.S(n), U.ptr(l2), U.ptr(f2), U.nthreads())
    assert U.bit_equal(l1, l2).all() and (f1 == f2).all()
    js = [np.empty((n, 9)) for _ in range(6)]
    P.orc_jacobians(U.ptr(a), U.S(n), *(U.ptr(j) for j in js[:3]))
    R.ref_jacobians(U.ptr(a), U.S(n), *(U.ptr(j) for j in js[3:]), U.nthreads())
    for k in range(3):
        assert U.bit_equal(js[k], js[k + 3]).all()


def test_port_generate_case_reproduces_perf_matrix():
    """generate_case(D2, U1, 1e-14) is the paper's perf matrix (bench.cpp:69-75,
    test_bench.cpp:62-74); its invariants carry the Appendix B bits."""
    out = np.empty((1, 9))
    d = np.array([1e-14])
    U.port().orc_generate_case(1, 1, U.ctypes_double(1e-3), U.ptr(d), U.S(1), U.ptr(out))
    assert U.bit_equal(out[0], U.perf_matrix()).all()


def test_port_generate_case_equals_compiled_reference_mat3():
    """The port's generate_case (src/bench.cpp:53-75) equals the compiled
    reference's own mat3 arithmetic over the same glue (ref_generate_case)."""
    deltas = np.array([10.0 ** (-k / 4.0) for k in range(4, 65)] + [0.0, 1e-14, 0.5, 3.0])
    R = U.ref()
    for gamma in (1e-3, 0.75, -2.5):
        for pi in (0, 1):
            for ki in (0, 1, 2):
                want = np.empty((deltas.size, 9))
                got = np.empty((deltas.size, 9))
                assert R.ref_generate_case(pi, ki, U.ctypes_double(gamma), U.ptr(deltas), U.S(deltas.size),
                                           U.ptr(want)) == 0
                U.port().orc_generate_case(pi, ki, U.ctypes_double(gamma), U.ptr(deltas), U.S(deltas.size),
                                           U.ptr(got))
                assert U.bit_equal(got, want).all(), (pi, ki, gamma)
