// Builds against include/eig33/batch.hpp and runs the batched C++ API on the
// GPU (tests/test_parity_gpu.py links it with _eig33cuda.so); checks a few
// known answers from the reference tests and prints "OK".
#include <cmath>
#include <cstdio>
#include <vector>

#include "eig33/batch.hpp"

int main() {
  std::vector<eig33::Mat3> a(3);
  a[0].e = {-1, 0, 0, 0, 1, 0, 0, 0, 2};  // acceptance C1
  a[1].e = {0, -1, 0, 1, 0, 0, 0, 0, 1};  // rotation: disc = -16, advisory
  a[2].e = {7.25, 0, 0, 0, 7.25, 0, 0, 0, 7.25};
  std::vector<eig33::InvariantSet> inv(3);
  eig33::invariants(a.data(), a.size(), inv.data());
  std::vector<eig33::EigenTriple> t(3);
  eig33::eigvals(a.data(), a.size(), t.data());
  bool ok = inv[0].disc == 36.0 && inv[0].i1 == 2.0 && inv[1].disc == -16.0 &&
            t[1].non_real_advisory && !t[0].non_real_advisory && t[2].lambda1 == 7.25 &&
            t[2].lambda3 == 7.25 && std::fabs(t[0].lambda3 - 2.0) < 1e-14;
  bool threw = false;
  try {
    eig33::eigvalss(a.data() + 1, 1, t.data());
  } catch (const eig33::NotSymmetric&) {
    threw = true;
  }
  ok = ok && threw;
  // the batched throw names the first record that fails the gate
  // (src/eigensolver.cpp:102 throws for exactly that record)
  std::vector<eig33::Mat3> s(5);
  for (auto& m : s) m.e = {2, 1, 0, 1, 3, -1, 0, -1, 4};
  s[3].e[1] = 1.5;
  s[4].e[2] = 0.5;
  std::vector<eig33::EigenTriple> st(5);
  std::size_t bad_at = 99;
  try {
    eig33::eigvalss(s.data(), s.size(), st.data());
  } catch (const eig33::NotSymmetricAt& e) {
    bad_at = e.index;
  }
  ok = ok && bad_at == 3 && std::fabs(st[0].lambda2 - 3.0) < 1e-14;
  // the study variants go through the same batched overload (invariants.hpp:74)
  std::vector<eig33::InvariantSet> nv(3), tv(3);
  eig33::invariants(a.data(), a.size(), nv.data(), eig33::AlgorithmVariant::Naive);
  eig33::invariants(a.data(), a.size(), tv.data(), eig33::AlgorithmVariant::NaiveTensor);
  ok = ok && nv[0].variant == eig33::AlgorithmVariant::Naive &&
       tv[0].variant == eig33::AlgorithmVariant::NaiveTensor && nv[0].i1 == 2.0 &&
       std::fabs(nv[0].j2 - 7.0 / 3.0) < 1e-14 && std::fabs(tv[0].j3 + 20.0 / 27.0) < 1e-14 &&
       std::fabs(nv[0].disc - 36.0) < 1e-12;
  std::printf("%s\n", ok ? "OK" : "FAIL");
  return ok ? 0 : 1;
}
