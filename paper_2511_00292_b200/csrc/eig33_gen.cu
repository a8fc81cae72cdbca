// eig33_gen.cu -- on-device synthetic corpora for the five BASELINE configs
// (recipes in eig33_gen_core.h, shared bit for bit with the host regeneration
// oracle/corpus_host.cpp) and the paper's accuracy-sweep corpora.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/eig33_cuda.h"
#include "eig33_gen_core.h"
#include "eig33_internal.h"

namespace eig33b {
namespace gen {

using eig33gen::M3;
using eig33gen::diag;
using eig33gen::similar;

__global__ void k_generate(int config, uint64_t seed, uint64_t first, long long n, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const M3 a = eig33gen::make_record(config, seed, first + (uint64_t)i);
#pragma unroll
    for (int k = 0; k < 9; ++k) out[i * 9 + k] = a.e[k];
  }
}

}  // namespace gen
}  // namespace eig33b

extern "C" int eig33cu_generate(int config, uint64_t seed, uint64_t first_index, size_t n,
                                double* d_a, void* stream) {
  eig33b::set_error("");
  if (n == 0) return EIG33_OK;
  if (config < 1 || config > 5 || !d_a) {
    eig33b::set_error("eig33cu_generate: bad argument");
    return EIG33_EINVAL;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = (long long)((n + 255) / 256);
  const long long grid = blocks < 16LL * sms ? blocks : 16LL * sms;
  eig33b::gen::k_generate<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(config, seed, first_index,
                                                                          (long long)n, d_a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    eig33b::set_error(std::string("k_generate launch: ") + cudaGetErrorString(e));
    return EIG33_ECUDA;
  }
  return EIG33_OK;
}

// ---------------------------------------------------------------------------
// The paper's accuracy-sweep corpora: generate_case(path,
// transform, delta) = (U * diag(low, 1, 1 + delta)) * inverse_adjugate(U),
// reference proj/src/bench.cpp:53-75, one record per delta.
//   path: 0 = D1 (low = 1), 1 = D2 (low = -1)
//   kind: 0 = Symm, 1 = U1, 2 = U2(gamma)
// ---------------------------------------------------------------------------
namespace eig33b {
namespace gen {

__device__ M3 make_transform(int kind, double gamma) {
  const double q = 0x1.6a09e667f3bcdp-1;  // fl(sqrt 2)/2, bench.cpp:56
  if (kind == 0) return {{q, -0.5, 0.5, q, 0.5, -0.5, 0.0, q, q}};
  if (kind == 1) return {{1, -1, 1, 1, 1, 1, -1, -1, 1}};
  return {{1, 1, 1, 1, 0, 1, 2, 1, 2.0 + gamma}};
}

__global__ void k_generate_case(int path, int kind, double gamma, const double* __restrict__ deltas,
                                long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const M3 u = make_transform(kind, gamma);
    const double low = path == 0 ? 1.0 : -1.0;
    const M3 a = similar(u, diag(low, 1.0, 1.0 + deltas[i]));
#pragma unroll
    for (int k = 0; k < 9; ++k) out[i * 9 + k] = a.e[k];
  }
}

}  // namespace gen
}  // namespace eig33b

extern "C" int eig33cu_generate_case(int path, int kind, double gamma, const double* d_deltas,
                                     size_t n, double* d_a, void* stream) {
  eig33b::set_error("");
  if (n == 0) return EIG33_OK;
  if (path < 0 || path > 1 || kind < 0 || kind > 2 || !d_deltas || !d_a ||
      (kind == 2 && gamma == 0.0)) {
    eig33b::set_error("eig33cu_generate_case: bad argument (gamma must be nonzero for U2)");
    return EIG33_EINVAL;
  }
  const long long blocks = (long long)((n + 255) / 256);
  const unsigned grid = (unsigned)(blocks < 4096 ? blocks : 4096);
  eig33b::gen::k_generate_case<<<grid, 256, 0, (cudaStream_t)stream>>>(path, kind, gamma, d_deltas,
                                                                      (long long)n, d_a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    eig33b::set_error(std::string("k_generate_case launch: ") + cudaGetErrorString(e));
    return EIG33_ECUDA;
  }
  return EIG33_OK;
}
