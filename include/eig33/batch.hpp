// eig33/batch.hpp -- batched overloads of the reference's C++ entry points,
// running on the B200 through the C ABI (include/eig33_cuda.h).
//
// Drop-in: a translation unit that already includes the reference headers
// (eig33/mat3.hpp, eig33/invariants.hpp, eig33/eigensolver.hpp from
// /root/reference/proj/include) gets these overloads next to the scalar ones:
//
//   eig33::invariants(const Mat3*, n, InvariantSet*, AlgorithmVariant = Stable)
//       batches  InvariantSet invariants(const Mat3&, AlgorithmVariant)  invariants.hpp:74
//   eig33::eigvals(const Mat3*, n, EigenTriple*)
//       batches  EigenTriple eigvals(const Mat3&)                        eigensolver.hpp:39
//   eig33::eigvalss(const Mat3*, n, EigenTriple*)   throws NotSymmetricAt (a NotSymmetric
//                                                   carrying the first bad index)
//       batches  EigenTriple eigvalss(const Mat3&)                       eigensolver.hpp:45
//   eig33::eigvals_packed(const Mat3*, n, double* lam, double* inv)   packed 24 B / 32 B outputs
//
// Without the reference headers on the include path, layout-identical
// stand-in types are declared (Mat3 = 72-B row-major record, mat3.hpp:24-28;
// InvariantSet 40 B, invariants.hpp:20-26; EigenTriple 32 B, eigensolver.hpp:29-34).
// All three AlgorithmVariants run on the GPU (Stable on the fused hot path,
// Naive / NaiveTensor on the study kernels), bit-exact like the scalar calls.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "eig33_cuda.h"

#if __has_include("eig33/mat3.hpp") && __has_include("eig33/invariants.hpp") && \
    __has_include("eig33/eigensolver.hpp") && !defined(EIG33_STANDALONE_TYPES)
#include "eig33/eigensolver.hpp"
#include "eig33/invariants.hpp"
#include "eig33/mat3.hpp"
#else
#include <array>
namespace eig33 {
struct Mat3 {
  std::array<double, 9> e{};
};
enum class AlgorithmVariant { Stable, Naive, NaiveTensor };
struct InvariantSet {
  double i1 = 0, j2 = 0, j3 = 0, disc = 0;
  AlgorithmVariant variant = AlgorithmVariant::Stable;
};
struct EigenTriple {
  double lambda1 = 0, lambda2 = 0, lambda3 = 0;
  bool non_real_advisory = false;
};
struct NotSymmetric : std::domain_error {
  NotSymmetric() : std::domain_error("matrix is not symmetric to working accuracy") {}
};
}  // namespace eig33
#endif

namespace eig33 {

static_assert(sizeof(Mat3) == 9 * sizeof(double), "Mat3 must be the 72-byte row-major record");

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// What the batched eigvalss throws: the reference's NotSymmetric (catchable as
// such, same what()), plus the index of the first record that failed the gate
// -- the record on which a loop of scalar eigvalss calls would have thrown
// (src/eigensolver.cpp:102).
struct NotSymmetricAt : NotSymmetric {
  std::size_t index;
  explicit NotSymmetricAt(std::size_t i) : NotSymmetric(), index(i) {}
};

namespace batch_detail {
inline void check(int rc) {
  if (rc == EIG33_OK) return;
  const std::string msg = eig33cu_last_error();
  if (rc == EIG33_ENOTSYM) {
    const long long i = eig33cu_last_notsym_index();
    throw NotSymmetricAt(i < 0 ? 0 : static_cast<std::size_t>(i));
  }
  if (rc == EIG33_EINVAL) throw std::invalid_argument(msg);
  throw CudaError(msg);
}
inline int device() { return 0; }
}  // namespace batch_detail

// Packed fast path: lam n x 3, inv n x 4 (nullable), flags n (nullable).
inline void eigvals_packed(const Mat3* a, std::size_t n, double* lam, double* inv = nullptr,
                           std::uint8_t* flags = nullptr) {
  batch_detail::check(eig33_eigvals_host(reinterpret_cast<const double*>(a), n, inv, lam, flags,
                                         batch_detail::device()));
}

inline void invariants(const Mat3* a, std::size_t n, InvariantSet* out,
                       AlgorithmVariant v = AlgorithmVariant::Stable) {
  std::vector<double> inv(n * 4);
  const int variant = v == AlgorithmVariant::Stable ? 0 : v == AlgorithmVariant::Naive ? 1 : 2;
  batch_detail::check(eig33_invariants_variant_host(reinterpret_cast<const double*>(a), n, variant,
                                                    inv.data(), batch_detail::device()));
  for (std::size_t i = 0; i < n; ++i) {
    out[i].i1 = inv[4 * i];
    out[i].j2 = inv[4 * i + 1];
    out[i].j3 = inv[4 * i + 2];
    out[i].disc = inv[4 * i + 3];
    out[i].variant = v;
  }
}

inline void eigvals(const Mat3* a, std::size_t n, EigenTriple* out) {
  std::vector<double> lam(n * 3);
  std::vector<std::uint8_t> flags(n);
  eigvals_packed(a, n, lam.data(), nullptr, flags.data());
  for (std::size_t i = 0; i < n; ++i) {
    out[i].lambda1 = lam[3 * i];
    out[i].lambda2 = lam[3 * i + 1];
    out[i].lambda3 = lam[3 * i + 2];
    out[i].non_real_advisory = (flags[i] & EIG33_FLAG_ADVISORY) != 0;
  }
}

// Throws NotSymmetricAt (a NotSymmetric) naming the first record that fails the
// gate; the outputs of every other record are written.
inline void eigvalss(const Mat3* a, std::size_t n, EigenTriple* out) {
  std::vector<double> lam(n * 3);
  std::vector<std::uint8_t> flags(n);
  const int rc = eig33_eigvalss_host(reinterpret_cast<const double*>(a), n, nullptr, lam.data(),
                                     flags.data(), batch_detail::device());
  for (std::size_t i = 0; i < n; ++i) {
    out[i].lambda1 = lam[3 * i];
    out[i].lambda2 = lam[3 * i + 1];
    out[i].lambda3 = lam[3 * i + 2];
    out[i].non_real_advisory = false;
  }
  batch_detail::check(rc);
}

}  // namespace eig33
