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
// path: 0 = dispatch like the kernel (moderate fast path when is_moderate),
//       1 = always the checked general path, 2 = always the moderate path
static bool moderate(const double* m) { return is_moderate(m) || is_moderate_or_zero(m); }
static Inv inv_path(const double* m, int path) {
  if (path == 2 || (path == 0 && moderate(m))) return invariants_moderate(m);
  return invariants(m);
}
static Lam lam_path(const double* m, const Inv& v, int path) {
  if (path == 2 || (path == 0 && moderate(m)))
    return from_invariants_moderate(m, v, eig33_tab);
  return from_invariants(m, v, eig33_tab);
}
// the always-valid CSE DAG of the invariants (identities 1-3, checked divisions)
void hm_invariants_dag(const double* a, size_t n, double* inv) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = invariants_dag(a + 9 * i);
    inv[4 * i] = v.i1; inv[4 * i + 1] = v.j2; inv[4 * i + 2] = v.j3; inv[4 * i + 3] = v.disc;
  }
}
// the general tier: invariants_dag + eig_general_bl (branch-light checked forms)
void hm_eigvals_general(const double* a, size_t n, double* lam) {
  for (size_t i = 0; i < n; ++i) {
    const double* m = a + 9 * i;
    const Inv v = invariants_dag(m);
    const Carry c{v.i1, v.j2, v.j3, v.disc, m[0], m[4], m[8]};
    const Lam l = eig_general_bl(c, eig33_tab);
    lam[3 * i] = l.l1; lam[3 * i + 1] = l.l2; lam[3 * i + 2] = l.l3;
  }
}
void hm_atan2_any(const double* y, const double* x, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = atan2_any(y[i], x[i], eig33_tab);
}
int hm_is_moderate(const double* a) { return is_moderate(a) ? 1 : 0; }
int hm_is_moderate_or_zero(const double* a) { return is_moderate_or_zero(a) ? 1 : 0; }
// path 3: the kernel's steady-state block (eig_fast) where its preconditions
// hold (moderate, j2 > 0, disc > 0), else path 0
void hm_eigvals_fast(const double* a, size_t n, double* lam) {
  for (size_t i = 0; i < n; ++i) {
    const double* m = a + 9 * i;
    Lam l;
    if (moderate(m)) {
      const Inv v = invariants_moderate(m);
      const Carry c{v.i1, v.j2, v.j3, v.disc, m[0], m[4], m[8]};
      l = fast_carry(v) ? eig_fast(c, eig33_tab) : eig_moderate_bl(c, eig33_tab);
    } else {
      l = from_invariants(m, invariants(m), eig33_tab);
    }
    lam[3 * i] = l.l1; lam[3 * i + 1] = l.l2; lam[3 * i + 2] = l.l3;
  }
}
void hm_invariants_path(const double* a, size_t n, double* inv, int path) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = inv_path(a + 9 * i, path);
    inv[4 * i] = v.i1; inv[4 * i + 1] = v.j2; inv[4 * i + 2] = v.j3; inv[4 * i + 3] = v.disc;
  }
}
void hm_eigvals_path(const double* a, size_t n, double* lam, int path) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = inv_path(a + 9 * i, path);
    const Lam l = lam_path(a + 9 * i, v, path);
    lam[3 * i] = l.l1; lam[3 * i + 1] = l.l2; lam[3 * i + 2] = l.l3;
  }
}
void hm_invariants(const double* a, size_t n, double* inv) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = inv_path(a + 9 * i, 0);
    inv[4 * i] = v.i1; inv[4 * i + 1] = v.j2; inv[4 * i + 2] = v.j3; inv[4 * i + 3] = v.disc;
  }
}
void hm_eigvals(const double* a, size_t n, double* lam, uint8_t* adv) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v = inv_path(a + 9 * i, 0);
    const Lam l = lam_path(a + 9 * i, v, 0);
    lam[3 * i] = l.l1; lam[3 * i + 1] = l.l2; lam[3 * i + 2] = l.l3;
    if (adv) adv[i] = advisory(a + 9 * i, v) ? 1 : 0;
  }
}
// the advisory decision for given invariants (i1 unused): the product's
// (certified squared comparison, reference-order fallback) and the
// reference-order one; and the reference-order tolerance itself
void hm_advisory2(const double* a, const double* inv, size_t n, uint8_t* fast, uint8_t* ref) {
  for (size_t i = 0; i < n; ++i) {
    const Inv v{inv[4 * i], inv[4 * i + 1], inv[4 * i + 2], inv[4 * i + 3]};
    fast[i] = advisory(a + 9 * i, v) ? 1 : 0;
    ref[i] = advisory_ref_order(a + 9 * i, v) ? 1 : 0;
  }
}
void hm_disc_tolerance(const double* a, const double* inv, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = disc_tolerance(a + 9 * i, inv[4 * i + 1], inv[4 * i + 2]);
}
void hm_atan2(const double* y, const double* x, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = atan2_pos(y[i], x[i], eig33_tab);
}
void hm_triple_angle(const double* j3, const double* disc, size_t n, double* out) {
  for (size_t i = 0; i < n; ++i) out[i] = triple_angle(j3[i], disc[i], eig33_tab);
}
void hm_sincos(const double* th, size_t n, double* s, double* c) {
  for (size_t i = 0; i < n; ++i) sincos_small(th[i], eig33_tab, s + i, c + i);
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

extern "C" {
void hm_invariants_variant(const double* a, size_t n, int v, double* inv) {
  for (size_t i = 0; i < n; ++i) {
    const Inv s = invariants_variant(a + 9 * i, v);
    inv[4 * i] = s.i1; inv[4 * i + 1] = s.j2; inv[4 * i + 2] = s.j3; inv[4 * i + 3] = s.disc;
  }
}
void hm_jacobians(const double* a, size_t n, double* jj2, double* jj3, double* jdisc) {
  for (size_t i = 0; i < n; ++i) {
    const double* m = a + 9 * i;
    jacobian_j2(m, jj2 + 9 * i);
    jacobian_j3(m, jj3 + 9 * i);
    const Inv s = invariants(m);
    jacobian_disc(m, s.j2, s.j3, jdisc + 9 * i);
  }
}
}
