"""CPU checks of the PRODUCT arithmetic (paper_2511_00292_b200/csrc/eig33_math.cuh
compiled for the host by tests/hostmath): the same source the sm_100a kernels
are built from, using only IEEE +,-,*,/,sqrt and explicit fma, so these
properties carry over to the device (re-checked on the GPU in test_parity_gpu).
"""
import ctypes

import mpmath
import numpy as np
import pytest

from tests import _util as U


def _call_unary(name, x, *extra):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    getattr(U.hostmath(), name)(U.ptr(x), U.S(x.size), *extra, U.ptr(out))
    return out


@pytest.mark.parametrize("c", [3, 6, 27])
def test_const_division_is_ieee(c):
    rng = np.random.default_rng(c)
    n = 1 << 21
    with np.errstate(all="ignore"):
        x = rng.standard_normal(n) * np.ldexp(1.0, rng.integers(-1074, 1024, n))
    tiny = np.ldexp(rng.random(1 << 16) + 1, rng.integers(-1074, -940, 1 << 16))
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                         1.7976931348623157e308, -1.7976931348623157e308, 3.0, 27.0, 1.0])
    # short mantissas: many exact quotients and quotients with few significant bits
    short = np.ldexp(rng.integers(1, 1 << 20, n).astype(np.float64) * (1 - 2 * rng.integers(0, 2, n)),
                     rng.integers(-960, 1000, n))
    x = np.concatenate([x, tiny, -tiny, specials, short, 3.0 * short])
    q = _call_unary("hm_div", x, ctypes.c_int(c))
    assert U.bit_equal(q, x / c).all()


def _libm_atan2(y, x):
    out = np.empty_like(y)
    U.hostmath().hm_libm_atan2(U.ptr(y), U.ptr(x), U.S(y.size), U.ptr(out))
    return out


def _atan2(y, x):
    out = np.empty_like(y)
    U.hostmath().hm_atan2(U.ptr(y), U.ptr(x), U.S(y.size), U.ptr(out))
    return out


def test_atan2_special_values_match_glibc():
    inf, nan = np.inf, np.nan
    ys = np.array([0.0, 0.0, 0.0, 0.0, 1.0, 1.0, inf, inf, inf, 1.0, 1.0, 0.0, 5e-324, 1e-310, 1e300,
                   1e-300, 1e308, 3.0])
    xs = np.array([0.0, -0.0, 2.0, -2.0, 0.0, -0.0, inf, -inf, 1.0, inf, -inf, nan, 1e300, -1e-310,
                   1e-300, -1e308, 1e-300, 3.0])
    assert U.bit_equal(_atan2(ys, xs), _libm_atan2(ys, xs)).all()


def test_atan2_correctly_rounded_and_within_1ulp_of_glibc():
    rng = np.random.default_rng(5)
    n = 1 << 21
    y = np.abs(rng.standard_normal(n)) * np.exp(rng.uniform(-30, 30, n))
    x = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    ours, gl = _atan2(y, x), _libm_atan2(y, x)
    d = np.abs(ours.view(np.int64) - gl.view(np.int64))
    assert d.max() <= 1
    assert (d == 0).mean() > 0.999
    mpmath.mp.prec = 200
    sample = np.concatenate([np.nonzero(d)[0][:100], rng.integers(0, n, 300)])
    wrong = sum(float(mpmath.atan2(mpmath.mpf(y[i]), mpmath.mpf(x[i]))) != ours[i] for i in sample)
    assert wrong <= 2  # correctly rounded except within ~2^-17 ulp of a midpoint


def test_sincos_correctly_rounded_on_0_pi3():
    rng = np.random.default_rng(6)
    n = 1 << 21
    th = rng.uniform(0, 1.0471975511965976, n)
    th[:4096] = rng.uniform(0, 1e-3, 4096)
    th[4096:4100] = [0.0, 1.0471975511965976, 5e-324, 2.0 ** -30]
    s = np.empty(n); c = np.empty(n); gs = np.empty(n); gc = np.empty(n)
    U.hostmath().hm_sincos(U.ptr(th), U.S(n), U.ptr(s), U.ptr(c))
    U.hostmath().hm_libm_sincos(U.ptr(th), U.S(n), U.ptr(gs), U.ptr(gc))
    for ours, gl in ((s, gs), (c, gc)):
        d = np.abs(ours.view(np.int64) - gl.view(np.int64))
        assert d.max() <= 1 and (d == 0).mean() > 0.997
    mpmath.mp.prec = 200
    wrong = 0
    for i in rng.integers(0, n, 400):
        wrong += float(mpmath.sin(mpmath.mpf(th[i]))) != s[i]
        wrong += float(mpmath.cos(mpmath.mpf(th[i]))) != c[i]
    assert wrong <= 1
    nan_s = np.empty(1); nan_c = np.empty(1)
    U.hostmath().hm_sincos(U.ptr(np.array([np.nan])), U.S(1), U.ptr(nan_s), U.ptr(nan_c))
    assert np.isnan(nan_s[0]) and np.isnan(nan_c[0])


def test_product_math_parity_vs_checker():
    a = U.mixed_corpus(1 << 19, 11)
    n = a.shape[0]
    inv = np.empty((n, 4))
    U.hostmath().hm_invariants(U.ptr(a), U.S(n), U.ptr(inv))
    assert U.bit_equal(inv, U.checker_invariants(a)).all()
    lam = np.empty((n, 3)); adv = np.empty(n, np.uint8)
    U.hostmath().hm_eigvals(U.ptr(a), U.S(n), U.ptr(lam), U.ptr(adv))
    lam_r, adv_r = U.checker_eigvals(a)
    assert (adv == adv_r).all()
    _, err, _ = U.lam_gate(a, lam, lam_r)
    assert (err == 0).mean() > 0.995


def test_product_study_variants_bitwise():
    a = U.mixed_corpus(1 << 16, 29)
    n = a.shape[0]
    H, R = U.hostmath(), U.ref()
    for v in (1, 2):
        x, y = np.empty((n, 4)), np.empty((n, 4))
        H.hm_invariants_variant(U.ptr(a), U.S(n), v, U.ptr(x))
        R.ref_invariants_variant(U.ptr(a), U.S(n), v, U.ptr(y), U.nthreads())
        assert U.bit_equal(x, y).all()
    js = [np.empty((n, 9)) for _ in range(6)]
    H.hm_jacobians(U.ptr(a), U.S(n), *(U.ptr(j) for j in js[:3]))
    R.ref_jacobians(U.ptr(a), U.S(n), *(U.ptr(j) for j in js[3:]), U.nthreads())
    for k in range(3):
        assert U.bit_equal(js[k], js[k + 3]).all()


def test_moderate_tier_with_exact_zeros_is_bitwise():
    """The moderate CSE/guard-free tier admits exact zeros (a zero is a multiple
    of every grain): sparse, diagonal, exact-repeated and near-identity records
    forced through it reproduce the reference bits."""
    rng = np.random.default_rng(41)
    n = 1 << 18
    a = rng.standard_normal((n, 9))
    a[rng.random((n, 9)) < 0.35] = 0.0                      # sparse
    a[: n // 8, [1, 2, 3, 5, 6, 7]] = 0.0                    # diagonal
    a[n // 8: n // 4] = np.round(a[n // 8: n // 4] * 64) / 64  # grid, ties, cancellations
    b = a[n // 4: n // 2]                                    # symmetric, some zeros
    b[:, [3, 6, 7]] = b[:, [1, 2, 5]]
    a = np.ascontiguousarray(a)
    H = U.hostmath()
    ok = np.array([H.hm_is_moderate_or_zero(U.ptr(a[i])) for i in range(0, n, 997)])
    assert ok.mean() > 0.95
    inv = np.empty((n, 4))
    H.hm_invariants(U.ptr(a), U.S(n), U.ptr(inv))  # dispatches like the kernel
    assert U.bit_equal(inv, U.checker_invariants(a)).all()
    lam = np.empty((n, 3))
    H.hm_eigvals_fast(U.ptr(a), U.S(n), U.ptr(lam))
    lam_r, _ = U.checker_eigvals(a, adv=False)
    U.lam_gate(a, lam, lam_r)


def _moderate_edge_corpus(n, seed):
    """Records at the edges of the moderate range [2^-100, 2^100): grid records
    (ties, exact cancellations, repeated eigenvalues) scaled to sit just inside
    either end, and near-scalar records c*I + d*E with off-diagonals down to
    ~2^-99 (differences and products land on the finest grains the range allows)."""
    rng = np.random.default_rng(seed)
    k = n // 4
    g = np.round(rng.uniform(-8, 8, (2 * k, 9)) * 64) / 64          # multiples of 2^-6, |.| <= 8
    g[g == 0] = 2.0 ** -6
    lo = g[:k] * 2.0 ** rng.integers(-93, -88, (k, 1))                # entries in [2^-99, 2^-85]
    hi = g[k:] * 2.0 ** rng.integers(88, 96, (k, 1))                  # entries in [2^82, 2^99]
    c = rng.uniform(-1, 1, (k, 1))
    d = 2.0 ** rng.uniform(-97, -60, (k, 1))
    e = rng.standard_normal((k, 9))
    e = np.where(np.abs(e) < 2.0 ** -2, 2.0 ** -2, e)
    ns = d * e
    ns[:, [0, 4, 8]] += c
    sym = ns.copy()
    sym[:, [3, 6, 7]] = sym[:, [1, 2, 5]]
    # finest grains: diagonals 2^-100 * (1 + i*2^-52) (differences of 2^-152),
    # off-diagonals 0 or +-2^-100 * small integers, and the mirror image at 2^99
    m = 4096
    x = 2.0 ** -100
    fine = np.zeros((m, 9))
    fine[:, 0] = x * (1 + rng.integers(0, 4, m) * 2.0 ** -52)
    fine[:, 4] = x * (1 + rng.integers(0, 4, m) * 2.0 ** -52)
    fine[:, 8] = x * (1 + rng.integers(0, 4, m) * 2.0 ** -52)
    off = rng.integers(-2, 3, (m, 6)) * x
    fine[:, [1, 2, 3, 5, 6, 7]] = off
    big = fine * 2.0 ** 198
    return np.ascontiguousarray(np.concatenate([lo, hi, ns, sym, fine, big])[-n:])


def test_widened_moderate_range_is_bitwise():
    """The moderate tier (guard-free CSE invariants, two-op divisions,
    guard-free eigenvalue stage) at the edges of [2^-100, 2^100) reproduces the
    compiled reference: invariants bit for bit, lambda within the gate."""
    a = _moderate_edge_corpus(1 << 18, 52)
    H = U.hostmath()
    ok = np.array([H.hm_is_moderate_or_zero(U.ptr(a[i])) for i in range(0, a.shape[0], 101)])
    assert ok.all()
    n = a.shape[0]
    inv = np.empty((n, 4))
    H.hm_invariants(U.ptr(a), U.S(n), U.ptr(inv))
    assert U.bit_equal(inv, U.checker_invariants(a)).all()
    lam = np.empty((n, 3))
    H.hm_eigvals_fast(U.ptr(a), U.S(n), U.ptr(lam))
    lam_r, _ = U.checker_eigvals(a, adv=False)
    U.lam_gate(a, lam, lam_r)
    # just outside the range the records must take the checked path
    out = a[:64] * 2.0 ** -20
    assert not any(H.hm_is_moderate_or_zero(U.ptr(out[i])) for i in range(64))


def test_transcendentals_misround_less_than_glibc():
    """Against mpmath (160 bits): our restricted-domain atan2 / sin / cos are
    correctly rounded on all but a tiny fraction of arguments, and misround
    less often than the glibc routines the reference calls."""
    mpmath.mp.prec = 160
    rng = np.random.default_rng(77)
    n = 8000
    th = rng.uniform(0, 1.0471975511965979, n)
    s, c, gs, gc = (np.empty(n) for _ in range(4))
    U.hostmath().hm_sincos(U.ptr(th), U.S(n), U.ptr(s), U.ptr(c))
    U.hostmath().hm_libm_sincos(U.ptr(th), U.S(n), U.ptr(gs), U.ptr(gc))
    y = np.abs(rng.standard_normal(n)) * np.exp(rng.uniform(-5, 5, n))
    x = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
    o, g = _atan2(y, x), _libm_atan2(y, x)
    ours = theirs = 0
    for i in range(n):
        t = mpmath.mpf(th[i])
        es, ec = float(mpmath.sin(t)), float(mpmath.cos(t))
        ea = float(mpmath.atan2(mpmath.mpf(y[i]), mpmath.mpf(x[i])))
        ours += (es != s[i]) + (ec != c[i]) + (ea != o[i])
        theirs += (es != gs[i]) + (ec != gc[i]) + (ea != g[i])
    assert ours <= 0.0005 * 3 * n
    assert ours < theirs


def test_invariants_dag_is_bitwise_for_any_record():
    """invariants_dag (gen_inv_dag.py, identities 1-3 only, checked divisions)
    reproduces the reference's invariants for every binary64 input: random bit
    patterns (inf, NaN, subnormals), 2^k-scaled records far outside the
    moderate range (overflow / underflow inside the DAG), zeros and ties."""
    rng = np.random.default_rng(2024)
    n = 1 << 17
    parts = [U.mixed_corpus(n, 5),
             rng.integers(0, 2 ** 64, size=(n, 9), dtype=np.uint64).view(np.float64),
             rng.standard_normal((n, 9)) * np.ldexp(1.0, rng.integers(-1074, 1000, size=(n, 1))),
             np.round(rng.standard_normal((n, 9)) * 2) * np.ldexp(1.0, rng.integers(-600, 600, size=(n, 1)))]
    with np.errstate(all="ignore"):
        a = np.ascontiguousarray(np.concatenate(parts))
    m = a.shape[0]
    inv = np.empty((m, 4))
    U.hostmath().hm_invariants_dag(U.ptr(a), U.S(m), U.ptr(inv))
    same = U.bit_equal(inv, U.checker_invariants(a)).all(axis=1)
    assert same.all(), f"{(~same).sum()} records differ, first {np.nonzero(~same)[0][:5]}"


def _adversarial(n, seed):
    rng = np.random.default_rng(seed)
    parts = [U.mixed_corpus(n, seed),
             rng.integers(0, 2 ** 64, size=(n, 9), dtype=np.uint64).view(np.float64),
             rng.standard_normal((n, 9)) * np.ldexp(1.0, rng.integers(-1074, 1000, size=(n, 1))),
             np.round(rng.standard_normal((n, 9)) * 2) * np.ldexp(1.0, rng.integers(-600, 600, size=(n, 1)))]
    with np.errstate(all="ignore"):
        return np.ascontiguousarray(np.concatenate(parts))


def test_general_tier_equals_checked_path():
    """The general tier's branch-light forms (invariants_dag + eig_general_bl:
    atan2_any, sqrt_any, selects for the j2 <= 0 collapse) give exactly the
    checked path's bits (invariants + from_invariants) on every input class."""
    a = _adversarial(1 << 16, 77)
    n = a.shape[0]
    H = U.hostmath()
    got, want = np.empty((n, 3)), np.empty((n, 3))
    H.hm_eigvals_general(U.ptr(a), U.S(n), U.ptr(got))
    H.hm_eigvals_path(U.ptr(a), U.S(n), U.ptr(want), 1)
    same = U.bit_equal(got, want).all(axis=1)
    assert same.all(), f"{(~same).sum()} records differ, first {np.nonzero(~same)[0][:5]}"


def test_atan2_any_equals_atan2_pos():
    rng = np.random.default_rng(3)
    n = 1 << 18
    y = np.abs(rng.integers(0, 2 ** 64, size=n, dtype=np.uint64).view(np.float64))
    x = rng.integers(0, 2 ** 64, size=n, dtype=np.uint64).view(np.float64)
    y[np.isnan(y)] = np.inf
    sp = np.array([0.0, np.inf, 1.0, 5e-324, 1e300, 2.0 ** -1000])
    y[: 36] = np.repeat(sp, 6)
    x[: 36] = np.tile(np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -3.0]), 6)
    H = U.hostmath()
    got, want = np.empty(n), np.empty(n)
    H.hm_atan2_any(U.ptr(y), U.ptr(x), U.S(n), U.ptr(got))
    H.hm_atan2(U.ptr(y), U.ptr(x), U.S(n), U.ptr(want))
    assert U.bit_equal(got, want).all()


def test_tiny_constant_division_is_ieee():
    """The constant divisions' tiny-operand form (x scaled by 2^120, the two-op
    quotient, rounding to the subnormal grid with the exact-midpoint repair;
    eig33_math.cuh div_tiny_fix) equals IEEE x/c for c = 3, 6, 27 on every
    binade below 2^-963, subnormals, and short mantissas (exact ties for c = 6)."""
    rng = np.random.default_rng(5)
    n = 1 << 20
    x = rng.integers(1, 60 << 52, size=n, dtype=np.int64).view(np.float64) * np.where(rng.random(n) < 0.5, -1, 1)
    y = np.ldexp(rng.integers(0, 1 << 20, size=n).astype(np.float64), rng.integers(-1074, -990, size=n))
    z = np.concatenate([x, y, -y, [0.0, -0.0, 5e-324, -5e-324, 3 * 5e-324, 6 * 5e-324, 9 * 5e-324,
                                   27 * 5e-324, 2.2250738585072014e-308, 2.0 ** -963, -(2.0 ** -963)]])
    for c in (3, 6, 27):
        out = np.empty_like(z)
        U.hostmath().hm_div(U.ptr(z), U.S(z.size), c, U.ptr(out))
        bad = ~U.bit_equal(out, z / c)
        assert not bad.any(), (c, z[bad][:5])


def _advisory2(a, inv):
    a = np.ascontiguousarray(a, dtype=np.float64)
    inv = np.ascontiguousarray(inv, dtype=np.float64)
    n = a.shape[0]
    fast, ref = np.empty(n, np.uint8), np.empty(n, np.uint8)
    U.hostmath().hm_advisory2(U.ptr(a), U.ptr(inv), U.S(n), U.ptr(fast), U.ptr(ref))
    return fast, ref


def test_advisory_certified_decision_equals_reference_order():
    """advisory() decides x = -disc vs the tolerance T by a squared comparison
    without the two square roots (eig33_math.cuh) and falls back to the
    reference-order T only near a tie: same flag as the reference-order form
    on the advisory-heavy configs, adversarial inputs, and on synthetic
    invariants placed within a few ulps of the tie (disc = -T (1 + k 2^-52))."""
    parts = [U.host_corpus(4, 1 << 17, 104), U.host_corpus(5, 1 << 17, 105),
             U.host_corpus(5, 1 << 15, 105, first=3 << 20), _adversarial(1 << 14, 91)]
    a = np.concatenate(parts)
    inv = U.checker_invariants(a)
    fast, ref = _advisory2(a, inv)
    assert (fast == ref).all(), np.nonzero(fast != ref)[0][:5]
    _, adv_r = U.checker_eigvals(a)
    assert (fast == adv_r).all()
    assert fast.sum() > 1000  # the flag-set branch is exercised
    # near-tie invariants on the records with a finite, normal tolerance
    n = a.shape[0]
    T = np.empty(n)
    U.hostmath().hm_disc_tolerance(U.ptr(a), U.ptr(inv), U.S(n), U.ptr(T))
    ok = np.isfinite(T) & (T > 1e-290) & (T < 1e290)
    at, it, Tt = a[ok][:20000], inv[ok][:20000], T[ok][:20000]
    for k in (-3, -1, 0, 1, 3, 1 << 6, 1 << 9, 1 << 12):
        it2 = it.copy()
        it2[:, 3] = -(Tt * (1.0 + k * 2.0 ** -52))
        f2, r2 = _advisory2(at, it2)
        assert (f2 == r2).all(), (k, np.nonzero(f2 != r2)[0][:5])
        if k == 0:
            assert not r2.any()  # disc == -T is not flagged
        if k >= 1:
            assert r2.all()
    # neighbours of the tie in ulp steps of disc itself
    for s in (-2, -1, 1, 2):
        it2 = it.copy()
        it2[:, 3] = -np.nextafter(Tt, np.inf if s > 0 else 0.0)
        if abs(s) == 2:
            it2[:, 3] = -np.nextafter(-it2[:, 3], np.inf if s > 0 else 0.0)
        f2, r2 = _advisory2(at, it2)
        assert (f2 == r2).all()
