/*
 * eig33_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library
 * (paper_2511_00292_b200/csrc) never links, calls or falls back to it.
 *
 * It restates, operation by operation, the reference's stable invariant
 * kernels and eigenvalue stage for one 72-byte row-major fp64 record and
 * loops that over a batch (the reference has no batch API).  Pinned by
 * tests/test_oracle.py against (1) the compiled reference core in
 * oracle/_ref/ (bitwise, random + edge corpora), (2) the KATs of the
 * reference's own tests, (3) the golden fixtures produced by the compiled
 * reference (tests/golden/make_golden.py writes the fixtures).
 *
 * Must be compiled with -ffp-contract=off (reference proj/src/CMakeLists.txt:9-10):
 * every written operation rounds once, no fused multiply-add.
 *
 * Reference line citations are relative to /root/reference/proj.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define ORC_EPS_MACH 0x1p-53 /* include/eig33/mat3.hpp:10 */

/* Row-major record accessor: e[3*i+j]  (include/eig33/mat3.hpp:24-28). */
#define E(m, i, j) ((m)[3 * (i) + (j)])

typedef struct {
  double d0, d1, d2;
} orc_ddiff;

/* src/invariants_impl.hpp:21-23 */
static orc_ddiff orc_diag_diff(const double *m) {
  orc_ddiff d;
  d.d0 = E(m, 0, 0) - E(m, 1, 1);
  d.d1 = E(m, 0, 0) - E(m, 2, 2);
  d.d2 = E(m, 1, 1) - E(m, 2, 2);
  return d;
}

/* src/invariants_impl.hpp:25 -- (a00 + a11) + a22 */
static double orc_i1(const double *m) { return (E(m, 0, 0) + E(m, 1, 1)) + E(m, 2, 2); }

/* src/invariants_impl.hpp:27-31 */
static double orc_j2(const double *m, orc_ddiff d) {
  double off = E(m, 0, 1) * E(m, 1, 0);
  off = off + E(m, 0, 2) * E(m, 2, 0);
  off = off + E(m, 1, 2) * E(m, 2, 1);
  double sq = d.d0 * d.d0;
  sq = sq + d.d1 * d.d1;
  sq = sq + d.d2 * d.d2;
  return sq / 6.0 + off;
}

/* src/invariants_impl.hpp:33-42 */
static double orc_j3(const double *m, orc_ddiff d) {
  const double t1 = d.d1 + d.d2;
  const double t2 = d.d0 - d.d2;
  const double t3 = (-d.d0) - d.d1;
  const double a01 = E(m, 0, 1), a02 = E(m, 0, 2), a10 = E(m, 1, 0);
  const double a12 = E(m, 1, 2), a20 = E(m, 2, 0), a21 = E(m, 2, 1);
  const double off = (a01 * a12) * a20 + (a02 * a10) * a21;
  double mixed = (a01 * a10) * t1;
  mixed = mixed + (a02 * a20) * t2;
  mixed = mixed + (a12 * a21) * t3;
  mixed = mixed / 3.0;
  const double dg = ((t1 * t2) * t3) / 27.0;
  return (off + mixed) - dg;
}

/* The 14 difference polynomials, src/invariants_impl.hpp:54-73.  Products are
 * left-associative, terms are summed in printed order.  r[9] follows the code
 * (+ m02*m21*d2, :67), not the paper's Algorithm 8 (which prints a minus). */
static void orc_dx(double x01, double x02, double x10, double x12, double x20, double x21,
                   orc_ddiff d, double r[14]) {
  const double d0 = d.d0, d1 = d.d1, d2 = d.d2;
  r[0] = ((x01 * x12) * x20) - ((x02 * x10) * x21);
  r[1] = ((((-x01) * x02) * d2) + ((x01 * x01) * x12)) - ((x02 * x02) * x21);
  r[2] = (((x01 * x21) * d1) - ((x01 * x01) * x20)) + ((x02 * x21) * x21);
  r[3] = (((x02 * x12) * d0) + ((x01 * x12) * x12)) - ((x02 * x02) * x10);
  r[4] = (((x01 * x12) * d1) - ((x01 * x02) * x10)) + ((x02 * x12) * x21);
  r[5] = (((x02 * x21) * d0) - ((x01 * x02) * x20)) + ((x01 * x12) * x21);
  r[6] = ((((-x02) * x10) * d2) + ((x01 * x10) * x12)) - ((x02 * x12) * x20);
  r[7] = ((((x12 * d0) * d1) - ((x02 * x10) * d1)) + ((x01 * x10) * x12)) - ((x12 * x12) * x21);
  r[8] = ((((x12 * d0) * d1) - ((x02 * x10) * d0)) + ((x02 * x12) * x20)) - ((x12 * x12) * x21);
  r[9] = ((((x01 * d1) * d2) + ((x02 * x21) * d2)) + ((x01 * x02) * x20)) - ((x01 * x01) * x10);
  r[10] = ((((x01 * d1) * d2) + ((x02 * x21) * d1)) + ((x01 * x12) * x21)) - ((x01 * x01) * x10);
  r[11] = (((((-x02) * d0) * d2) + ((x01 * x12) * d0)) + ((x02 * x12) * x21)) - ((x02 * x02) * x20);
  r[12] = ((((x02 * d0) * d2) + ((x01 * x12) * d2)) - ((x01 * x02) * x10)) + ((x02 * x02) * x20);
  r[13] = ((((d0 * d1) * d2) - ((x01 * x10) * d0)) + ((x02 * x20) * d1)) - ((x12 * x21) * d2);
}

/* src/invariants_impl.hpp:75 */
static const double orc_w[14] = {9, 6, 6, 6, 8, 8, 8, 2, 2, 2, 2, 2, 2, 1};

/* src/invariants_impl.hpp:77-85: u from A, v from A^T (argument mirroring),
 * acc starts at +0.0 and adds (w*u)*v in k order. */
static double orc_disc(const double *m, orc_ddiff d) {
  double u[14], v[14];
  orc_dx(E(m, 0, 1), E(m, 0, 2), E(m, 1, 0), E(m, 1, 2), E(m, 2, 0), E(m, 2, 1), d, u);
  orc_dx(E(m, 1, 0), E(m, 2, 0), E(m, 0, 1), E(m, 2, 1), E(m, 0, 2), E(m, 1, 2), d, v);
  double acc = 0.0;
  for (int k = 0; k < 14; ++k) acc = acc + (orc_w[k] * u[k]) * v[k];
  return acc;
}

/* ---- mat3 helpers on the advisory path (src/mat3.cpp) ---- */

/* src/mat3.cpp:7 and :9-16 */
static void orc_dev(const double *m, double *s) {
  const double mean = ((E(m, 0, 0) + E(m, 1, 1)) + E(m, 2, 2)) / 3.0;
  memcpy(s, m, 9 * sizeof(double));
  s[0] = m[0] - mean;
  s[4] = m[4] - mean;
  s[8] = m[8] - mean;
}

/* src/mat3.cpp:32-47 */
static void orc_cofactor(const double *m, double *c) {
  const double a00 = m[0], a01 = m[1], a02 = m[2];
  const double a10 = m[3], a11 = m[4], a12 = m[5];
  const double a20 = m[6], a21 = m[7], a22 = m[8];
  c[0] = a11 * a22 - a12 * a21;
  c[1] = a12 * a20 - a10 * a22;
  c[2] = a10 * a21 - a11 * a20;
  c[3] = a02 * a21 - a01 * a22;
  c[4] = a00 * a22 - a02 * a20;
  c[5] = a01 * a20 - a00 * a21;
  c[6] = a01 * a12 - a02 * a11;
  c[7] = a02 * a10 - a00 * a12;
  c[8] = a00 * a11 - a01 * a10;
}

/* src/mat3.cpp:66-70 -- sum of squares from +0.0 in row-major order. */
static double orc_frob(const double *m) {
  double s = 0.0;
  for (int k = 0; k < 9; ++k) s = s + m[k] * m[k];
  return sqrt(s);
}

/* src/invariants.cpp:64-74 (jacobian_disc) feeding src/eigensolver.cpp:45-47
 * (disc_tolerance).  j2/j3 are the public stable wrappers: same values as the
 * inlined kernels (invariants.cpp:19,36). */
static double orc_disc_tolerance(const double *m) {
  const orc_ddiff d = orc_diag_diff(m);
  const double j2 = orc_j2(m, d);
  const double j3 = orc_j3(m, d);
  const double c2 = (12.0 * j2) * j2;
  const double c3 = 54.0 * j3;
  double dv[9], cd[9], g[9], jd[9];
  orc_dev(m, dv);
  orc_cofactor(dv, cd);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) g[3 * i + j] = c2 * E(m, j, i) - c3 * cd[3 * i + j];
  orc_dev(g, jd);
  return 10.0 * ((orc_frob(jd) * orc_frob(dv)) * ORC_EPS_MACH);
}

/* src/eigensolver.cpp:32-34 */
static double orc_diag_mean(const double *m) {
  return m[0] + ((m[4] - m[0]) + (m[8] - m[0])) / 3.0;
}

/* src/eigensolver.cpp:84-89 */
double orc_triple_angle(double j3, double disc) {
  const double dc = disc > 0.0 ? disc : 0.0;
  return atan2(sqrt(27.0 * dc), 27.0 * j3);
}

/* fl(sqrt(3))/2, src/eigensolver.cpp:16 */
static const double orc_root3_half = 0x1.bb67ae8584caap-1;

/* src/eigensolver.cpp:49-80 (from_invariants) + :36-40 (sort3).  adv may be
 * NULL, in which case the advisory (which never changes lambda, :54) is
 * skipped. */
static void orc_from_invariants(const double *m, double i1, double j2, double j3, double disc,
                                double *lam, uint8_t *adv) {
  if (adv) *adv = (disc < 0.0) ? (uint8_t)(disc < -orc_disc_tolerance(m)) : 0;
  if (j2 <= 0.0) {
    const double mu = orc_diag_mean(m);
    lam[0] = lam[1] = lam[2] = mu;
    return;
  }
  const double phi = orc_triple_angle(j3, disc);
  const double r = 2.0 * sqrt(3.0 * j2);
  double sn, cs;
  sincos(phi / 3.0, &sn, &cs);
  const double ch = -0.5 * cs;
  const double sh = orc_root3_half * sn;
  double x = (i1 + r * (ch - sh)) / 3.0;
  double y = (i1 + r * (ch + sh)) / 3.0;
  double z = (i1 + r * cs) / 3.0;
  double t;
  if (y < x) { t = x; x = y; y = t; }
  if (z < y) { t = y; y = z; z = t; }
  if (y < x) { t = x; x = y; y = t; }
  lam[0] = x;
  lam[1] = y;
  lam[2] = z;
}

/* ---- batch entry points (ctypes) ---- */

/* invariants(a, Stable) over a batch: src/invariants.cpp:76-85 -> n x {i1,j2,j3,disc}. */
void orc_invariants(const double *a, size_t n, double *inv) {
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    const orc_ddiff d = orc_diag_diff(m);
    inv[4 * i + 0] = orc_i1(m);
    inv[4 * i + 1] = orc_j2(m, d);
    inv[4 * i + 2] = orc_j3(m, d);
    inv[4 * i + 3] = orc_disc(m, d);
  }
}

/* eigvals over a batch: src/eigensolver.cpp:91-95.  inv/adv nullable. */
void orc_eigvals(const double *a, size_t n, double *inv, double *lam, uint8_t *adv) {
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    const orc_ddiff d = orc_diag_diff(m);
    const double i1 = orc_i1(m), j2 = orc_j2(m, d), j3 = orc_j3(m, d), disc = orc_disc(m, d);
    if (inv) {
      inv[4 * i + 0] = i1;
      inv[4 * i + 1] = j2;
      inv[4 * i + 2] = j3;
      inv[4 * i + 3] = disc;
    }
    orc_from_invariants(m, i1, j2, j3, disc, lam + 3 * i, adv ? adv + i : NULL);
  }
}

/* eigvalss over a batch: src/eigensolver.cpp:97-117.  status[i] = 1 where the
 * scalar API would throw NotSymmetric (lambda left as NaN), else 0. */
void orc_eigvalss(const double *a, size_t n, double *inv, double *lam, uint8_t *status) {
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    double maxabs = 0.0;
    for (int k = 0; k < 9; ++k) maxabs = fmax(maxabs, fabs(m[k]));
    const double asym = fmax(fmax(fabs(m[1] - m[3]), fabs(m[2] - m[6])), fabs(m[5] - m[7]));
    if (asym > (4.0 * ORC_EPS_MACH) * maxabs) {
      if (status) status[i] = 1;
      lam[3 * i] = lam[3 * i + 1] = lam[3 * i + 2] = NAN;
      if (inv) inv[4 * i] = inv[4 * i + 1] = inv[4 * i + 2] = inv[4 * i + 3] = NAN;
      continue;
    }
    if (status) status[i] = 0;
    double s[9];
    memcpy(s, m, sizeof s);
    s[3] = m[1];
    s[6] = m[2];
    s[7] = m[5];
    const orc_ddiff d = orc_diag_diff(s);
    const double i1 = orc_i1(s), j2 = orc_j2(s, d), j3 = orc_j3(s, d), disc = orc_disc(s, d);
    if (inv) {
      inv[4 * i + 0] = i1;
      inv[4 * i + 1] = j2;
      inv[4 * i + 2] = j3;
      inv[4 * i + 3] = disc;
    }
    orc_from_invariants(s, i1, j2, j3, disc, lam + 3 * i, NULL);
  }
}

/* triple_angle over a batch (include/eig33/eigensolver.hpp:21). */
void orc_triple_angle_batch(const double *j3, const double *disc, size_t n, double *phi) {
  for (size_t i = 0; i < n; ++i) phi[i] = orc_triple_angle(j3[i], disc[i]);
}

/* Advisory-only pass (src/eigensolver.cpp:54): adv[i] = disc < -tol(A). */
void orc_advisory(const double *a, size_t n, uint8_t *adv) {
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    const orc_ddiff d = orc_diag_diff(m);
    const double disc = orc_disc(m, d);
    adv[i] = (disc < 0.0) ? (uint8_t)(disc < -orc_disc_tolerance(m)) : 0;
  }
}

/* ---- threaded streaming driver (cpu_baseline, kind "port") ---- */

typedef struct {
  const double *a;
  double *inv, *lam;
  size_t lo, hi;
} orc_job;

static void *orc_worker(void *p) {
  orc_job *j = (orc_job *)p;
  orc_eigvals(j->a + 9 * j->lo, j->hi - j->lo, j->inv ? j->inv + 4 * j->lo : NULL,
              j->lam + 3 * j->lo, NULL);
  return NULL;
}

/* Contiguous shards, one pthread each.  Returns 0. */
int orc_eigvals_mt(const double *a, size_t n, double *inv, double *lam, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  orc_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].a = a;
    jobs[t].inv = inv;
    jobs[t].lam = lam;
    jobs[t].lo = n * (size_t)t / (size_t)nthreads;
    jobs[t].hi = n * (size_t)(t + 1) / (size_t)nthreads;
    pthread_create(&th[t], NULL, orc_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* ---- accuracy-study variants ---- */

/* src/invariants.cpp:21-28 */
static double orc_j2_naive(const double *m) {
  const double a00 = m[0], a01 = m[1], a02 = m[2], a10 = m[3], a11 = m[4], a12 = m[5];
  const double a20 = m[6], a21 = m[7], a22 = m[8];
  return (a00 * a00 - a00 * a11 - a00 * a22 + 3.0 * a01 * a10 + 3.0 * a02 * a20 + a11 * a11 -
          a11 * a22 + 3.0 * a12 * a21 + a22 * a22) /
         3.0;
}

/* src/invariants.cpp:38-52 */
static double orc_j3_naive(const double *m) {
  const double a00 = m[0], a01 = m[1], a02 = m[2], a10 = m[3], a11 = m[4], a12 = m[5];
  const double a20 = m[6], a21 = m[7], a22 = m[8];
  double s = 2.0 * a00 * a00 * a00;
  s -= 3.0 * a00 * a00 * a11;
  s -= 3.0 * a00 * a00 * a22;
  s += 9.0 * a00 * a01 * a10;
  s += 9.0 * a00 * a02 * a20;
  s -= 3.0 * a00 * a11 * a11;
  s += 12.0 * a00 * a11 * a22;
  s -= 18.0 * a00 * a12 * a21;
  s -= 3.0 * a00 * a22 * a22;
  s += 9.0 * a01 * a10 * a11;
  s -= 18.0 * a01 * a10 * a22;
  s += 27.0 * a01 * a12 * a20;
  s += 27.0 * a02 * a10 * a21;
  s -= 18.0 * a02 * a11 * a20;
  s += 9.0 * a02 * a20 * a22;
  s += 2.0 * a11 * a11 * a11;
  s -= 3.0 * a11 * a11 * a22;
  s += 9.0 * a11 * a12 * a21;
  s -= 3.0 * a11 * a22 * a22;
  s += 9.0 * a12 * a21 * a22;
  s += 2.0 * a22 * a22 * a22;
  return s / 27.0;
}

/* src/invariants.cpp:30-34 with matmul/trace, src/mat3.cpp:7,18-26 */
static double orc_j2_tensor(const double *m) {
  double d[9];
  orc_dev(m, d);
  double t[3];
  for (int i = 0; i < 3; ++i)
    t[i] = d[3 * i] * d[i] + d[3 * i + 1] * d[3 + i] + d[3 * i + 2] * d[6 + i];
  return (t[0] + t[1] + t[2]) / 2.0;
}

/* src/invariants.cpp:54 with det, src/mat3.cpp:49-55 */
static double orc_j3_tensor(const double *m) {
  double d[9];
  orc_dev(m, d);
  return d[0] * (d[4] * d[8] - d[5] * d[7]) - d[1] * (d[3] * d[8] - d[5] * d[6]) +
         d[2] * (d[3] * d[7] - d[4] * d[6]);
}

/* src/invariants.cpp:58 */
static double orc_disc_naive(double j2, double j3) { return 4.0 * j2 * j2 * j2 - 27.0 * j3 * j3; }

/* invariants(a, v), src/invariants.cpp:76-98: v = 0 Stable, 1 Naive, 2 NaiveTensor */
void orc_invariants_variant(const double *a, size_t n, int v, double *inv) {
  if (v == 0) {
    orc_invariants(a, n, inv);
    return;
  }
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    const double j2 = v == 1 ? orc_j2_naive(m) : orc_j2_tensor(m);
    const double j3 = v == 1 ? orc_j3_naive(m) : orc_j3_tensor(m);
    inv[4 * i + 0] = orc_i1(m);
    inv[4 * i + 1] = j2;
    inv[4 * i + 2] = j3;
    inv[4 * i + 3] = orc_disc_naive(j2, j3);
  }
}

/* eigvals_naive, src/eigensolver.cpp:119-123 */
void orc_eigvals_naive(const double *a, size_t n, double *lam, uint8_t *adv) {
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    const double j2 = orc_j2_naive(m), j3 = orc_j3_naive(m);
    orc_from_invariants(m, orc_i1(m), j2, j3, orc_disc_naive(j2, j3), lam + 3 * i,
                        adv ? adv + i : NULL);
  }
}

/* jacobian_j2 / j3 / disc, src/invariants.cpp:60-74; each output n x 9, nullable */
void orc_jacobians(const double *a, size_t n, double *jj2, double *jj3, double *jdisc) {
  for (size_t i = 0; i < n; ++i) {
    const double *m = a + 9 * i;
    double dv[9], cd[9], g[9];
    orc_dev(m, dv);
    if (jj2)
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) jj2[9 * i + 3 * r + c] = dv[3 * c + r];
    if (jj3) {
      orc_cofactor(dv, cd);
      orc_dev(cd, jj3 + 9 * i);
    }
    if (jdisc) {
      const orc_ddiff d = orc_diag_diff(m);
      const double j2 = orc_j2(m, d), j3 = orc_j3(m, d);
      const double c2 = (12.0 * j2) * j2, c3 = 54.0 * j3;
      orc_cofactor(dv, cd);
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) g[3 * r + c] = c2 * m[3 * c + r] - c3 * cd[3 * r + c];
      orc_dev(g, jdisc + 9 * i);
    }
  }
}

/* ---- paper corpora: make_transform / generate_case (src/bench.cpp:53-75) ---- */

/* src/mat3.cpp:18-26 */
static void orc_matmul(const double *a, const double *b, double *c) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

/* src/mat3.cpp:49-64 (transpose of the cofactor matrix over det) */
static void orc_inverse_adjugate(const double *a, double *inv) {
  const double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                     a[2] * (a[3] * a[7] - a[4] * a[6]);
  double c[9];
  orc_cofactor(a, c);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) inv[3 * i + j] = c[3 * j + i] / det;
}

/* path 0 = D1, 1 = D2; kind 0 = Symm, 1 = U1, 2 = U2(gamma); one record per delta */
void orc_generate_case(int path, int kind, double gamma, const double *deltas, size_t n,
                       double *out) {
  const double q = 0x1.6a09e667f3bcdp-1; /* std::numbers::sqrt2_v<double> / 2.0 */
  double u[9];
  if (kind == 0) {
    const double s[9] = {q, -0.5, 0.5, q, 0.5, -0.5, 0.0, q, q};
    memcpy(u, s, sizeof u);
  } else if (kind == 1) {
    const double s[9] = {1, -1, 1, 1, 1, 1, -1, -1, 1};
    memcpy(u, s, sizeof u);
  } else {
    const double s[9] = {1, 1, 1, 1, 0, 1, 2, 1, 2.0 + gamma};
    memcpy(u, s, sizeof u);
  }
  double uinv[9], ud[9];
  orc_inverse_adjugate(u, uinv);
  for (size_t i = 0; i < n; ++i) {
    const double d[9] = {path == 0 ? 1.0 : -1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0 + deltas[i]};
    orc_matmul(u, d, ud);
    orc_matmul(ud, uinv, out + 9 * i);
  }
}
