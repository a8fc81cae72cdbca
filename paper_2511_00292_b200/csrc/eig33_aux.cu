// eig33_aux.cu -- batched accuracy-study entry points:
// the naive / tensor invariant variants, eigvals_naive, and the invariant
// Jacobians.  Not on the throughput path: one record per thread, grid-stride,
// direct loads; bit-exact against the reference like the hot path (compiled
// with --fmad=false).
#include <cuda_runtime.h>
#include <stdint.h>

#define EIG33_TABLE_DECL static __device__ __align__(16)  // as in eig33_kernels.cu
#include "eig33_tables.h"
#include "eig33_math.cuh"
#include "eig33_internal.h"
#include "../../include/eig33_cuda.h"

namespace eig33b {
namespace aux {

__device__ __forceinline__ void load9(const double* __restrict__ a, long long i, double m[9]) {
#pragma unroll
  for (int k = 0; k < 9; ++k) m[k] = __ldg(a + i * 9 + k);
}

__global__ void __launch_bounds__(256) k_inv_variant(const double* __restrict__ a, long long n,
                                                     int variant, double* __restrict__ inv) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double m[9];
    load9(a, i, m);
    const Inv v = invariants_variant(m, variant);
    inv[i * 4 + 0] = v.i1;
    inv[i * 4 + 1] = v.j2;
    inv[i * 4 + 2] = v.j3;
    inv[i * 4 + 3] = v.disc;
  }
}

// eigvals_naive (src/eigensolver.cpp:119-123): from_invariants on naive j2/j3,
// disc_naive, including the advisory (:54, tolerance from the stable kernels).
__global__ void __launch_bounds__(256) k_eig_naive(const double* __restrict__ a, long long n,
                                                   double* __restrict__ lam,
                                                   uint8_t* __restrict__ flags) {
  __shared__ __align__(16) double tab[EIG33_TAB_N + 7];
  copy_table(tab, eig33_tab);
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double m[9];
    load9(a, i, m);
    const Inv v = invariants_variant(m, 1);
    const Lam L = from_invariants(m, v, tab);
    lam[i * 3 + 0] = L.l1;
    lam[i * 3 + 1] = L.l2;
    lam[i * 3 + 2] = L.l3;
    if (flags) {
      bool adv = false;
      if (v.disc < 0.0) {
        const Inv s = invariants(m);
        adv = v.disc < -disc_tolerance(m, s.j2, s.j3);
      }
      flags[i] = adv ? EIG33_FLAG_ADVISORY : 0;
    }
  }
}

__global__ void __launch_bounds__(256) k_jacobians(const double* __restrict__ a, long long n,
                                                   double* __restrict__ jj2, double* __restrict__ jj3,
                                                   double* __restrict__ jdisc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double m[9], g[9];
    load9(a, i, m);
    if (jj2) {
      jacobian_j2(m, g);
#pragma unroll
      for (int k = 0; k < 9; ++k) jj2[i * 9 + k] = g[k];
    }
    if (jj3) {
      jacobian_j3(m, g);
#pragma unroll
      for (int k = 0; k < 9; ++k) jj3[i * 9 + k] = g[k];
    }
    if (jdisc) {
      const Inv s = invariants(m);
      jacobian_disc(m, s.j2, s.j3, g);
#pragma unroll
      for (int k = 0; k < 9; ++k) jdisc[i * 9 + k] = g[k];
    }
  }
}

// disc_naive(j2, j3) = ((4 j2) j2) j2 - (27 j3) j3 (src/invariants.cpp:58), elementwise
__global__ void __launch_bounds__(256) k_disc_naive(const double* __restrict__ j2,
                                                    const double* __restrict__ j3, long long n,
                                                    double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = disc_naive(j2[i], j3[i]);
}

static unsigned grid_for(size_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = (long long)((n + 255) / 256);
  return (unsigned)(blocks < 8LL * sms ? blocks : 8LL * sms);
}

static int done(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return EIG33_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return EIG33_ECUDA;
}

}  // namespace aux
}  // namespace eig33b

using namespace eig33b;

extern "C" {

int eig33cu_invariants_variant(const double* d_a, size_t n, int variant, double* d_inv,
                               void* stream) {
  set_error("");
  if (n == 0) return EIG33_OK;
  if (!d_a || !d_inv || variant < 0 || variant > 2) {
    set_error("eig33cu_invariants_variant: bad argument");
    return EIG33_EINVAL;
  }
  if (variant == 0) return eig33cu_invariants(d_a, n, d_inv, stream);
  aux::k_inv_variant<<<aux::grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_a, (long long)n, variant,
                                                                        d_inv);
  return aux::done("k_inv_variant launch");
}

int eig33cu_eigvals_naive(const double* d_a, size_t n, double* d_lam, uint8_t* d_flags,
                          void* stream) {
  set_error("");
  if (n == 0) return EIG33_OK;
  if (!d_a || !d_lam) {
    set_error("eig33cu_eigvals_naive: null pointer");
    return EIG33_EINVAL;
  }
  aux::k_eig_naive<<<aux::grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_a, (long long)n, d_lam,
                                                                      d_flags);
  return aux::done("k_eig_naive launch");
}

int eig33cu_jacobians(const double* d_a, size_t n, double* d_jj2, double* d_jj3, double* d_jdisc,
                      void* stream) {
  set_error("");
  if (n == 0) return EIG33_OK;
  if (!d_a || (!d_jj2 && !d_jj3 && !d_jdisc)) {
    set_error("eig33cu_jacobians: bad argument");
    return EIG33_EINVAL;
  }
  aux::k_jacobians<<<aux::grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_a, (long long)n, d_jj2,
                                                                      d_jj3, d_jdisc);
  return aux::done("k_jacobians launch");
}

int eig33cu_disc_naive(const double* d_j2, const double* d_j3, size_t n, double* d_disc,
                       void* stream) {
  set_error("");
  if (n == 0) return EIG33_OK;
  if (!d_j2 || !d_j3 || !d_disc) {
    set_error("eig33cu_disc_naive: null pointer");
    return EIG33_EINVAL;
  }
  aux::k_disc_naive<<<aux::grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_j2, d_j3, (long long)n,
                                                                       d_disc);
  return aux::done("k_disc_naive launch");
}

}  // extern "C"
