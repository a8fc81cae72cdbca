// hostmath.cpp -- TEST INFRASTRUCTURE: the product's per-record arithmetic
// (paper_2511_00292_b200/csrc/eig33_math.cuh) compiled for the CPU, so its
// numerics can be checked here, without a GPU, against glibc, mpmath and the
// compiled reference.  Never loaded by the product path.
#include <stddef.h>
#include <stdint.h>
#define EIG33_TABLE_DECL static const
#include "../../paper_2511_00292_b200/csrc/eig33_tables.h"
#include "../../paper_2511_00292_b200/csrc/eig33_math.cuh"

using namespace eig33b;

extern "C" {
void hm_invariants(const double* a, size_t n, double* inv) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = invariants(a + 9 * i);
    inv[4 * i] = v.i1; inv[4 * i + 1] = v.j2; inv[4 * i + 2] = v.j3; inv[4 * i + 3] = v.disc;
  }
}
void hm_eigvals(const double* a, size_t n, double* lam, uint8_t* adv) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = invariants(a + 9 * i);
    const Lam l = from_invariants(a + 9 * i, v, eig33_at_c, eig33_at_t, eig33_sc);
    lam[3 * i] = l.l1; lam[3 * i + 1] = l.l2; lam[3 * i + 2] = l.l3;
    if (adv) adv[i] = advisory(a + 9 * i, v) ? 1 : 0;
  }
}
void hm_atan2(const double* y, const double* x, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = atan2_pos(y[i], x[i], eig33_at_c, eig33_at_t);
}
void hm_triple_angle(const double* j3, const double* disc, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = triple_angle(j3[i], disc[i], eig33_at_c, eig33_at_t);
}
void hm_sincos(const double* th, size_t n, double* s, double* c) {
  for (size_t i = 0; i < n; ++i) sincos_small(th[i], eig33_sc, s + i, c + i);
}
void hm_div(const double* x, size_t n, int which, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = which == 3 ? div3(x[i]) : which == 6 ? div6(x[i]) : div27(x[i]);
}
}

// glibc reference calls (what the compiled reference links: atan2, sincos)
#include <math.h>
extern "C" {
void hm_libm_atan2(const double* y, const double* x, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = ::atan2(y[i], x[i]);
}
void hm_libm_sincos(const double* th, size_t n, double* s, double* c) {
  for (size_t i = 0; i < n; ++i) ::sincos(th[i], s + i, c + i);
}
}
