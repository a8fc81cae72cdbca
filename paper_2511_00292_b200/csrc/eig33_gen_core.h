// eig33_gen_core.h -- recipes of the synthetic corpora for the five BASELINE
// configs, written once for the device generator (eig33_gen.cu, nvcc
// --fmad=false) and the host regeneration used by bench.py's reference arm
// and the tests (oracle/corpus_host.cpp, g++ -ffp-contract=off).
//
// Bit-identical on both sides by construction: every floating-point value is
// produced by IEEE-754 binary64 +, -, *, / and sqrt (correctly rounded on
// both), integer operations, and exact conversions.  No libm / libdevice
// transcendental is called: log, cos(2*pi*u), 10^x are the polynomial
// evaluations below (accurate to a few ulp, which is all a synthetic
// distribution needs -- what matters is that both builds round the same
// operations the same way).  FMA contraction must be off in both builds.
//
// Counter-based: record i of config c with seed s depends only on (c, s, i),
// so any shard or sub-range regenerates independently.  Similarity products
// use the reference's association (V*D)*V^-1 with V^-1 = inverse_adjugate(V)
// (proj/src/bench.cpp:69-75, proj/src/mat3.cpp:20-26,49-64).
//
//   1  symmetric: A = (Q*diag(l))*Q^T, Q Haar (Gram-Schmidt of a Gaussian,
//      R_ii > 0), l_i ~ U[-1,1]; upper triangle mirrored so A is bitwise symmetric
//   2  coalescing: A = (V*diag(1,1+e,1+2e))*V^-1, V Haar, e = 10^-u, u ~ U[1,15]
//   3  throughput: A = (V*diag(l))*V^-1, V_ij ~ N(0,1) rejected unless
//      cond_2(V) <= 1e3, l_i ~ U[-10,10]
//   4  ill-conditioned: V = (U*diag(1,s,s^2))*W^T, U,W Haar, s = 10^-t, t ~ U[1,4];
//      l = (1, 1+e, 2), e = 10^-u, u ~ U[0,12]
//   5  edge/scaling, quarter = (i >> 20) & 3 (contiguous 2^20 blocks):
//      q0 near-scalar c*I + d*E (c ~ U[-1,1], E_ij ~ N(0,1), d = 10^-u, u ~ U[8,16]);
//      q1 exact repeated/triple: (U1*diag(x,x,y))*U1^-1, x,y in Z/64, |x|,|y| <= 16,
//         half with y = x; q2 diagonal (N(0,1), a quarter with a repeated entry);
//      q3 G_ij ~ N(0,1) scaled by 2^k, k ~ U{-500..500}
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define EIG33_GEN_HD __host__ __device__ inline
#else
#include <string.h>
#define EIG33_GEN_HD static inline
#endif

namespace eig33gen {

struct M3 {
  double e[9];
};

EIG33_GEN_HD double from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}
EIG33_GEN_HD uint64_t to_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
EIG33_GEN_HD double sqrt_(double x) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(x);
#else
  return __builtin_sqrt(x);
#endif
}
// 2^k for -1022 <= k <= 1023 (exact)
EIG33_GEN_HD double pow2i(int k) { return from_bits((uint64_t)(k + 1023) << 52); }

// ---- portable elementary functions (only +,-,*,/ and integer ops) ----
// natural log of x > 0 (normal): x = m 2^e, m in [sqrt(1/2), sqrt(2)),
// log x = e ln2 + 2 atanh(s), s = (m-1)/(m+1), |s| <= 0.1716, odd series to s^23.
EIG33_GEN_HD double log_p(double x) {
  const uint64_t b = to_bits(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = from_bits((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull);  // [1,2)
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  const double s = (m - 1.0) / (m + 1.0), s2 = s * s;
  double t = 1.0 / 23.0;
  t = t * s2 + 1.0 / 21.0;
  t = t * s2 + 1.0 / 19.0;
  t = t * s2 + 1.0 / 17.0;
  t = t * s2 + 1.0 / 15.0;
  t = t * s2 + 1.0 / 13.0;
  t = t * s2 + 1.0 / 11.0;
  t = t * s2 + 1.0 / 9.0;
  t = t * s2 + 1.0 / 7.0;
  t = t * s2 + 1.0 / 5.0;
  t = t * s2 + 1.0 / 3.0;
  t = t * s2 + 1.0;
  const double ln2_hi = 0.6931471805599453, ln2_lo = 2.3190468138462996e-17;
  return (double)e * ln2_hi + ((double)e * ln2_lo + 2.0 * s * t);
}
// sin and cos of x in [0, pi/4]: Taylor series to x^17 / x^16.
EIG33_GEN_HD void sincos_q(double x, double* s, double* c) {
  const double x2 = x * x;
  double sn = 1.0 / 355687428096000.0;   // 1/17!
  sn = sn * x2 - 1.0 / 1307674368000.0;  // 1/15!
  sn = sn * x2 + 1.0 / 6227020800.0;     // 1/13!
  sn = sn * x2 - 1.0 / 39916800.0;       // 1/11!
  sn = sn * x2 + 1.0 / 362880.0;         // 1/9!
  sn = sn * x2 - 1.0 / 5040.0;           // 1/7!
  sn = sn * x2 + 1.0 / 120.0;            // 1/5!
  sn = sn * x2 - 1.0 / 6.0;              // 1/3!
  *s = x + x * (x2 * sn);
  double cs = 1.0 / 20922789888000.0;    // 1/16!
  cs = cs * x2 - 1.0 / 87178291200.0;    // 1/14!
  cs = cs * x2 + 1.0 / 479001600.0;      // 1/12!
  cs = cs * x2 - 1.0 / 3628800.0;        // 1/10!
  cs = cs * x2 + 1.0 / 40320.0;          // 1/8!
  cs = cs * x2 - 1.0 / 720.0;            // 1/6!
  cs = cs * x2 + 1.0 / 24.0;             // 1/4!
  cs = cs * x2 - 0.5;                    // 1/2!
  *c = 1.0 + x2 * cs;
}
// cos(2 pi u) for u in [0, 1): octant reduction (exact: v = 8u), then the
// quarter-range series on (pi/4) f, f in [0, 1].
EIG33_GEN_HD double cos2pi(double u) {
  const double v = u * 8.0;                  // exact
  const int k = (int)v;                      // octant 0..7
  const double f = v - (double)k;            // exact, [0,1)
  const double pi4 = 0.7853981633974483;
  double s, c;
  // angle within the octant measured from the nearest multiple of pi/2
  const bool odd = (k & 1) != 0;
  sincos_q(pi4 * (odd ? (1.0 - f) : f), &s, &c);
  // 2 pi u = (pi/2) q + r, q = k >> 1; r = (pi/4) f, or pi/2 - (pi/4)(1-f) when odd
  const int q = k >> 1;
  const double cr = odd ? s : c;   // cos r
  const double sr = odd ? c : s;   // sin r
  switch (q & 3) {
    case 0: return cr;
    case 1: return -sr;
    case 2: return -cr;
    default: return sr;
  }
}
// 10^x for x in [-16, 0]: 2^y, y = x log2(10) = k + f, f in [0,1); 2^f = e^(f ln2)
// by its Taylor series to degree 20; result scaled by the exact 2^k.
EIG33_GEN_HD double exp10_p(double x) {
  const double y = x * 3.321928094887362;
  double kf = (double)(int64_t)y;
  if (kf > y) kf = kf - 1.0;  // floor
  const double g = (y - kf) * 0.6931471805599453;  // in [0, ln2)
  double t = 1.0 / 2432902008176640000.0;  // 1/20!
  t = t * g + 1.0 / 121645100408832000.0;  // 1/19!
  t = t * g + 1.0 / 6402373705728000.0;  // 1/18!
  t = t * g + 1.0 / 355687428096000.0;  // 1/17!
  t = t * g + 1.0 / 20922789888000.0;  // 1/16!
  t = t * g + 1.0 / 1307674368000.0;  // 1/15!
  t = t * g + 1.0 / 87178291200.0;  // 1/14!
  t = t * g + 1.0 / 6227020800.0;  // 1/13!
  t = t * g + 1.0 / 479001600.0;  // 1/12!
  t = t * g + 1.0 / 39916800.0;  // 1/11!
  t = t * g + 1.0 / 3628800.0;  // 1/10!
  t = t * g + 1.0 / 362880.0;  // 1/9!
  t = t * g + 1.0 / 40320.0;  // 1/8!
  t = t * g + 1.0 / 5040.0;  // 1/7!
  t = t * g + 1.0 / 720.0;  // 1/6!
  t = t * g + 1.0 / 120.0;  // 1/5!
  t = t * g + 1.0 / 24.0;  // 1/4!
  t = t * g + 1.0 / 6.0;  // 1/3!
  t = t * g + 1.0 / 2.0;  // 1/2!
  t = t * g + 1.0;  // 1/1!
  t = t * g + 1.0;  // 1/0!
  return t * pow2i((int)kf);
}

// ---- counter-based RNG ----
EIG33_GEN_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
struct Rng {
  uint64_t key;
  uint64_t ctr;
};
EIG33_GEN_HD Rng rng_make(uint64_t seed, int config, uint64_t idx, uint32_t attempt) {
  Rng r;
  r.key = mix64(seed ^ mix64(((uint64_t)config << 56) ^ idx ^ ((uint64_t)attempt << 40)));
  r.ctr = 0;
  return r;
}
EIG33_GEN_HD uint64_t rng_next(Rng& r) { return mix64(r.key + 0x9e3779b97f4a7c15ull * (++r.ctr)); }
EIG33_GEN_HD double rng_uniform(Rng& r) { return (double)(rng_next(r) >> 11) * 0x1p-53; }  // [0,1)
EIG33_GEN_HD double rng_uniform(Rng& r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }
// Box-Muller: sqrt(-2 log u1) cos(2 pi u2), u1 in (0,1)
EIG33_GEN_HD double rng_gauss(Rng& r) {
  const double u1 = ((double)(rng_next(r) >> 11) + 0.5) * 0x1p-53;
  const double u2 = rng_uniform(r);
  return sqrt_(-2.0 * log_p(u1)) * cos2pi(u2);
}

// ---- 3x3 algebra (reference association, no contraction) ----
EIG33_GEN_HD M3 matmul(const M3& a, const M3& b) {
  M3 c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c.e[3 * i + j] = (a.e[3 * i] * b.e[j] + a.e[3 * i + 1] * b.e[3 + j]) + a.e[3 * i + 2] * b.e[6 + j];
  return c;
}
EIG33_GEN_HD M3 transpose(const M3& a) {
  M3 t = {{a.e[0], a.e[3], a.e[6], a.e[1], a.e[4], a.e[7], a.e[2], a.e[5], a.e[8]}};
  return t;
}
EIG33_GEN_HD M3 cofactor(const M3& a) {
  M3 c;
  c.e[0] = a.e[4] * a.e[8] - a.e[5] * a.e[7];
  c.e[1] = a.e[5] * a.e[6] - a.e[3] * a.e[8];
  c.e[2] = a.e[3] * a.e[7] - a.e[4] * a.e[6];
  c.e[3] = a.e[2] * a.e[7] - a.e[1] * a.e[8];
  c.e[4] = a.e[0] * a.e[8] - a.e[2] * a.e[6];
  c.e[5] = a.e[1] * a.e[6] - a.e[0] * a.e[7];
  c.e[6] = a.e[1] * a.e[5] - a.e[2] * a.e[4];
  c.e[7] = a.e[2] * a.e[3] - a.e[0] * a.e[5];
  c.e[8] = a.e[0] * a.e[4] - a.e[1] * a.e[3];
  return c;
}
EIG33_GEN_HD double det(const M3& a) {
  return (a.e[0] * (a.e[4] * a.e[8] - a.e[5] * a.e[7]) - a.e[1] * (a.e[3] * a.e[8] - a.e[5] * a.e[6])) +
         a.e[2] * (a.e[3] * a.e[7] - a.e[4] * a.e[6]);
}
EIG33_GEN_HD M3 inverse_adjugate(const M3& a) {
  const double d = det(a);
  const M3 adj = transpose(cofactor(a));
  M3 r;
  for (int k = 0; k < 9; ++k) r.e[k] = adj.e[k] / d;
  return r;
}
EIG33_GEN_HD M3 diag(double a, double b, double c) {
  M3 d = {{a, 0, 0, 0, b, 0, 0, 0, c}};
  return d;
}
EIG33_GEN_HD M3 similar(const M3& v, const M3& d) { return matmul(matmul(v, d), inverse_adjugate(v)); }

// Haar-orthogonal Q: modified Gram-Schmidt on the columns of a Gaussian
// matrix (equivalent to QR with R_ii > 0).
EIG33_GEN_HD M3 haar(Rng& r) {
  double c[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) c[j][i] = rng_gauss(r);
  for (int j = 0; j < 3; ++j) {
    for (int k = 0; k < j; ++k) {
      const double p = c[j][0] * c[k][0] + c[j][1] * c[k][1] + c[j][2] * c[k][2];
      for (int i = 0; i < 3; ++i) c[j][i] -= p * c[k][i];
    }
    const double nrm = sqrt_(c[j][0] * c[j][0] + c[j][1] * c[j][1] + c[j][2] * c[j][2]);
    for (int i = 0; i < 3; ++i) c[j][i] /= nrm;
  }
  M3 q;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) q.e[3 * i + j] = c[j][i];
  return q;
}

// Is cond_2(V) <= kappa?  The extreme eigenvalues of the Gram matrix G = V^T V
// are found by Newton on its characteristic cubic p(t) = t^3 - c2 t^2 + c1 t - c0
// (three nonnegative real roots): from t = 0 the iterates rise monotonically to
// the smallest root, from t = tr G they fall to the largest; each loop stops
// when an iterate no longer moves in its direction (or after 100 steps).
EIG33_GEN_HD bool cond2_at_most(const M3& v, double kappa) {
  const M3 g = matmul(transpose(v), v);
  const double c2 = (g.e[0] + g.e[4]) + g.e[8];
  const double c1 = ((g.e[0] * g.e[4] - g.e[1] * g.e[3]) + (g.e[0] * g.e[8] - g.e[2] * g.e[6])) +
                    (g.e[4] * g.e[8] - g.e[5] * g.e[7]);
  const double c0 = det(g);
  if (!(c0 > 0.0)) return false;
  double lo = 0.0;
  for (int it = 0; it < 100; ++it) {
    const double p = ((lo - c2) * lo + c1) * lo - c0;
    const double dp = (3.0 * lo - 2.0 * c2) * lo + c1;
    const double nx = lo - p / dp;
    if (!(nx > lo)) break;
    lo = nx;
  }
  double hi = c2;
  for (int it = 0; it < 100; ++it) {
    const double p = ((hi - c2) * hi + c1) * hi - c0;
    const double dp = (3.0 * hi - 2.0 * c2) * hi + c1;
    const double nx = hi - p / dp;
    if (!(nx < hi)) break;
    hi = nx;
  }
  if (!(lo > 0.0)) return false;
  return hi <= (kappa * kappa) * lo;
}

// Record idx of config 1..5.
EIG33_GEN_HD M3 make_record(int config, uint64_t seed, uint64_t idx) {
  if (config == 1) {
    Rng r = rng_make(seed, 1, idx, 0);
    const M3 q = haar(r);
    const double l0 = rng_uniform(r, -1, 1), l1 = rng_uniform(r, -1, 1), l2 = rng_uniform(r, -1, 1);
    M3 a = matmul(matmul(q, diag(l0, l1, l2)), transpose(q));
    a.e[3] = a.e[1];
    a.e[6] = a.e[2];
    a.e[7] = a.e[5];
    return a;
  }
  if (config == 2) {
    Rng r = rng_make(seed, 2, idx, 0);
    const M3 v = haar(r);
    const double eps = exp10_p(-rng_uniform(r, 1, 15));
    return similar(v, diag(1.0, 1.0 + eps, 1.0 + 2.0 * eps));
  }
  if (config == 3) {
    for (uint32_t attempt = 0;; ++attempt) {
      Rng r = rng_make(seed, 3, idx, attempt);
      M3 v;
      for (int k = 0; k < 9; ++k) v.e[k] = rng_gauss(r);
      if (!cond2_at_most(v, 1e3) && attempt < 64) continue;
      const double l0 = rng_uniform(r, -10, 10), l1 = rng_uniform(r, -10, 10), l2 = rng_uniform(r, -10, 10);
      return similar(v, diag(l0, l1, l2));
    }
  }
  if (config == 4) {
    Rng r = rng_make(seed, 4, idx, 0);
    const M3 u = haar(r), w = haar(r);
    const double s = exp10_p(-rng_uniform(r, 1, 4));
    const M3 v = matmul(matmul(u, diag(1.0, s, s * s)), transpose(w));
    const double eps = exp10_p(-rng_uniform(r, 0, 12));
    return similar(v, diag(1.0, 1.0 + eps, 2.0));
  }
  // config 5
  Rng r = rng_make(seed, 5, idx, 0);
  const int quarter = (int)((idx >> 20) & 3);
  M3 a;
  if (quarter == 0) {
    const double c = rng_uniform(r, -1, 1);
    const double dl = exp10_p(-rng_uniform(r, 8, 16));
    for (int k = 0; k < 9; ++k) a.e[k] = dl * rng_gauss(r);
    a.e[0] += c;
    a.e[4] += c;
    a.e[8] += c;
  } else if (quarter == 1) {
    const M3 u1 = {{1, -1, 1, 1, 1, 1, -1, -1, 1}};
    const double x = (double)((int64_t)(rng_next(r) % 2049) - 1024) / 64.0;
    double y = (double)((int64_t)(rng_next(r) % 2049) - 1024) / 64.0;
    if (rng_next(r) & 1) y = x;
    a = similar(u1, diag(x, x, y));
  } else if (quarter == 2) {
    const double d0 = rng_gauss(r), d1 = rng_gauss(r);
    const double d2 = (rng_next(r) & 3) == 0 ? d0 : rng_gauss(r);
    a = diag(d0, d1, d2);
  } else {
    const int k = (int)(rng_next(r) % 1001) - 500;
    const double s = pow2i(k);  // exact scaling: N(0,1) * 2^k stays normal for |k| <= 500
    for (int j = 0; j < 9; ++j) a.e[j] = rng_gauss(r) * s;
  }
  return a;
}

}  // namespace eig33gen
