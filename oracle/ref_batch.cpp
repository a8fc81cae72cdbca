// ref_batch.cpp -- batch-over-records driver around the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY (checker + CPU baseline).  Linked by oracle/Makefile
// with /root/reference/proj/src/{mat3,invariants,eigensolver}.cpp compiled in
// place with the reference's own flags (-std=c++20 -O3 -ffp-contract=off,
// proj/src/CMakeLists.txt:5-10) into oracle/_ref/libeig33_ref.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// load it.  It calls the reference's public per-matrix API:
//   eig33::invariants(const Mat3&, AlgorithmVariant)  include/eig33/invariants.hpp:74
//   eig33::eigvals(const Mat3&)                       include/eig33/eigensolver.hpp:39
//   eig33::eigvalss(const Mat3&)                      include/eig33/eigensolver.hpp:45
//   eig33::triple_angle(double, double)               include/eig33/eigensolver.hpp:21
//   eig33::eigvals_checksum_loop(const Mat3&, n)      include/eig33/eigensolver.hpp:57
#include <pthread.h>
#include <sched.h>

#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "eig33/eigensolver.hpp"
#include "eig33/invariants.hpp"
#include "eig33/mat3.hpp"

namespace {

eig33::Mat3 load(const double* p) {
  eig33::Mat3 m;
  std::memcpy(m.e.data(), p, sizeof(double) * 9);
  return m;
}

// CPUs this process may run on, in order (the baseline pins thread t to the
// t-th of them: contiguous shards, one pinned thread per core).
std::vector<int> allowed_cpus() {
  std::vector<int> cpus;
  cpu_set_t set;
  CPU_ZERO(&set);
  if (sched_getaffinity(0, sizeof set, &set) == 0)
    for (int c = 0; c < CPU_SETSIZE; ++c)
      if (CPU_ISSET(c, &set)) cpus.push_back(c);
  return cpus;
}

template <class F>
void parallel_shards(std::size_t n, int nthreads, F&& body) {
  if (nthreads <= 1 || n < 2) {
    body(std::size_t{0}, n);
    return;
  }
  static const std::vector<int> cpus = allowed_cpus();
  std::vector<std::thread> pool;
  pool.reserve(nthreads);
  for (int t = 0; t < nthreads; ++t) {
    const std::size_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
    pool.emplace_back([&body, lo, hi] { body(lo, hi); });
    if (!cpus.empty()) {
      cpu_set_t one;
      CPU_ZERO(&one);
      CPU_SET(cpus[t % cpus.size()], &one);
      pthread_setaffinity_np(pool.back().native_handle(), sizeof one, &one);
    }
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// n x {i1, j2, j3, disc}
int ref_invariants(const double* a, std::size_t n, double* inv, int nthreads) {
  parallel_shards(n, nthreads, [=](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const auto s = eig33::invariants(load(a + 9 * i), eig33::AlgorithmVariant::Stable);
      inv[4 * i + 0] = s.i1;
      inv[4 * i + 1] = s.j2;
      inv[4 * i + 2] = s.j3;
      inv[4 * i + 3] = s.disc;
    }
  });
  return 0;
}

// n x {l1, l2, l3}; adv nullable (n bytes)
int ref_eigvals(const double* a, std::size_t n, double* lam, std::uint8_t* adv, int nthreads) {
  parallel_shards(n, nthreads, [=](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const auto t = eig33::eigvals(load(a + 9 * i));
      lam[3 * i + 0] = t.lambda1;
      lam[3 * i + 1] = t.lambda2;
      lam[3 * i + 2] = t.lambda3;
      if (adv) adv[i] = t.non_real_advisory ? 1 : 0;
    }
  });
  return 0;
}

// status[i] = 1 where eigvalss throws NotSymmetric (lambda = NaN there)
int ref_eigvalss(const double* a, std::size_t n, double* lam, std::uint8_t* status, int nthreads) {
  parallel_shards(n, nthreads, [=](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      try {
        const auto t = eig33::eigvalss(load(a + 9 * i));
        lam[3 * i + 0] = t.lambda1;
        lam[3 * i + 1] = t.lambda2;
        lam[3 * i + 2] = t.lambda3;
        if (status) status[i] = 0;
      } catch (const eig33::NotSymmetric&) {
        lam[3 * i + 0] = lam[3 * i + 1] = lam[3 * i + 2] = __builtin_nan("");
        if (status) status[i] = 1;
      }
    }
  });
  return 0;
}

int ref_triple_angle(const double* j3, const double* disc, std::size_t n, double* phi) {
  for (std::size_t i = 0; i < n; ++i) phi[i] = eig33::triple_angle(j3[i], disc[i]).phi;
  return 0;
}

std::uint64_t ref_checksum_loop(const double* a, std::uint64_t n) {
  return eig33::eigvals_checksum_loop(load(a), n);
}

}  // extern "C"

extern "C" {

// invariants(a, v) for v = 0 Stable, 1 Naive, 2 NaiveTensor (include/eig33/invariants.hpp:74)
int ref_invariants_variant(const double* a, std::size_t n, int v, double* inv, int nthreads) {
  const auto var = v == 0 ? eig33::AlgorithmVariant::Stable
                   : v == 1 ? eig33::AlgorithmVariant::Naive
                            : eig33::AlgorithmVariant::NaiveTensor;
  parallel_shards(n, nthreads, [=](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const auto s = eig33::invariants(load(a + 9 * i), var);
      inv[4 * i + 0] = s.i1;
      inv[4 * i + 1] = s.j2;
      inv[4 * i + 2] = s.j3;
      inv[4 * i + 3] = s.disc;
    }
  });
  return 0;
}

// eigvals_naive (include/eig33/eigensolver.hpp:49)
int ref_eigvals_naive(const double* a, std::size_t n, double* lam, std::uint8_t* adv, int nthreads) {
  parallel_shards(n, nthreads, [=](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const auto t = eig33::eigvals_naive(load(a + 9 * i));
      lam[3 * i + 0] = t.lambda1;
      lam[3 * i + 1] = t.lambda2;
      lam[3 * i + 2] = t.lambda3;
      if (adv) adv[i] = t.non_real_advisory ? 1 : 0;
    }
  });
  return 0;
}

// jacobian_j2 / jacobian_j3 / jacobian_disc (include/eig33/invariants.hpp:62-69)
int ref_jacobians(const double* a, std::size_t n, double* jj2, double* jj3, double* jdisc,
                  int nthreads) {
  parallel_shards(n, nthreads, [=](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const eig33::Mat3 m = load(a + 9 * i);
      if (jj2) std::memcpy(jj2 + 9 * i, eig33::jacobian_j2(m).e.data(), 72);
      if (jj3) std::memcpy(jj3 + 9 * i, eig33::jacobian_j3(m).e.data(), 72);
      if (jdisc) std::memcpy(jdisc + 9 * i, eig33::jacobian_disc(m).e.data(), 72);
    }
  });
  return 0;
}

}  // extern "C"

extern "C" {

// bench::generate_case (src/bench.cpp:69-75) for one path / transform over a
// vector of deltas.  bench.cpp itself needs GMP/MPFR/Boost headers absent here,
// so its two lines of glue are restated -- the transform constants of
// make_transform (src/bench.cpp:52-67) and matmul(matmul(u, d), uinv) -- while
// every rounded operation runs in the reference's own compiled mat3.cpp
// (Mat3::diagonal, matmul, inverse_adjugate; include/eig33/mat3.hpp:32,57,69).
// path: 0 = D1, 1 = D2; kind: 0 = Symm, 1 = U1, 2 = U2(gamma).
int ref_generate_case(int path, int kind, double gamma, const double* deltas, std::size_t n,
                      double* out) {
  constexpr double q = 0x1.6a09e667f3bcdp-1;  // std::numbers::sqrt2_v<double> / 2.0 (exact halving)
  eig33::Mat3 u;
  if (kind == 0) u = eig33::Mat3{{q, -0.5, 0.5, q, 0.5, -0.5, 0.0, q, q}};
  else if (kind == 1) u = eig33::Mat3{{1, -1, 1, 1, 1, 1, -1, -1, 1}};
  else if (gamma != 0.0) u = eig33::Mat3{{1, 1, 1, 1, 0, 1, 2, 1, 2.0 + gamma}};
  else return 2;
  const double low = path == 0 ? 1.0 : -1.0;
  const eig33::Mat3 uinv = eig33::inverse_adjugate(u);
  for (std::size_t i = 0; i < n; ++i) {
    const eig33::Mat3 d = eig33::Mat3::diagonal(low, 1.0, 1.0 + deltas[i]);
    const eig33::Mat3 a = eig33::matmul(eig33::matmul(u, d), uinv);
    std::memcpy(out + 9 * i, a.e.data(), 72);
  }
  return 0;
}

}  // extern "C"
