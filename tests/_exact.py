"""Exact-spectrum fallback judge for ill-conditioned eigenbases (config 4).

TEST INFRASTRUCTURE.  Restates the reference's exact oracle idea
(proj/src/oracle.cpp:98-105 char_poly on exact rationals, :237-278
spectrum_reference, :306-307 bound units) without GMP/MPFR: the input doubles
are exact dyadic rationals, the characteristic cubic is formed exactly with
fractions.Fraction, and its roots are resolved with mpmath at 400 bits.

Criterion (BASELINE north_star): where lambda_gpu fails the
4-ulp test against lambda_ref, accept it iff its forward error against the
exact spectrum, in units of b = kappa2(V)*||A||_F*2^-53, is no larger than the
reference's own.  The common factor b cancels in that comparison, so the test
is max_k |l_gpu,k - l_exact,k| <= max_k |l_ref,k - l_exact,k|.  For a complex
exact pair the real parts are used (the reference returns the clamped
projection there, eigensolver.hpp:24-28).
"""
from fractions import Fraction

import mpmath
import numpy as np


def _char_poly(a):
    m = [[Fraction(float(a[3 * i + j])) for j in range(3)] for i in range(3)]
    tr = m[0][0] + m[1][1] + m[2][2]
    minors = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) + (m[0][0] * m[2][2] - m[0][2] * m[2][0]) + (
        m[1][1] * m[2][2] - m[1][2] * m[2][1])
    det = (m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1])
           - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0])
           + m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]))
    return [Fraction(1), -tr, minors, -det]


def exact_spectrum(a):
    with mpmath.workprec(400):
        coeffs = [mpmath.mpf(c.numerator) / c.denominator for c in _char_poly(a)]
        roots = mpmath.polyroots(coeffs, maxsteps=400, extraprec=800)
        re = sorted(mpmath.re(r) for r in roots)
    return re


def within_reference_forward_error(a_rows, lam_gpu, lam_ref):
    ok = np.zeros(len(a_rows), dtype=bool)
    for i, (a, lg, lr) in enumerate(zip(a_rows, lam_gpu, lam_ref)):
        ex = exact_spectrum(a)
        with mpmath.workprec(400):
            eg = max(abs(mpmath.mpf(float(lg[k])) - ex[k]) for k in range(3))
            er = max(abs(mpmath.mpf(float(lr[k])) - ex[k]) for k in range(3))
        ok[i] = eg <= er
    return ok
