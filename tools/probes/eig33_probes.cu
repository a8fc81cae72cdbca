// eig33_probes.cu -- measurement library for bench.py and tools/ (NOT part of the product
// _eig33cuda.so or its C ABI):
// the achievable FP64-pipe issue rate of this GPU, used as the
// roofline denominator for the FP64-bound fused kernel.  MEASURED_PEAKS.json
// carries only HBM and bf16 peaks, so bench.py measures this on the box.
//
// Every thread runs 8 independent DFMA chains (enough ILP to cover the DFMA
// latency with 8 warps per SMSP); the result is written so nothing is dead.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
template <int OP>
__global__ void __launch_bounds__(256) k_dfma_rate(int iters, double seed, double* out) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed + (threadIdx.x + k) * 1e-9;
  const double m = 0.9999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = __fma_rn(x[k], m, c);
      if (OP == 1) x[k] = __dmul_rn(x[k], m);
      if (OP == 2) x[k] = __dadd_rn(x[k], c);
      if (OP == 3) x[k] = (k & 1) ? __dmul_rn(x[k], m) : __dadd_rn(x[k], c);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[blockIdx.x] = s;  // practically never taken; defeats DCE
}
}  // namespace

// Returns DFMA warp-instructions*32 (thread-level FP64 instructions) per
// second measured over `reps` launches, or a negative value on error.
template <int OP>
static double probe(int reps, int iters);
extern "C" double eig33_probe_fp64_rate(int reps) { return probe<0>(reps, 4096); }
// op: 0 DFMA, 1 DMUL, 2 DADD, 3 DMUL/DADD mix; iters scales the duration
extern "C" double eig33_probe_fp64_op(int op, int reps, int iters) {
  switch (op) {
    case 1: return probe<1>(reps, iters);
    case 2: return probe<2>(reps, iters);
    case 3: return probe<3>(reps, iters);
    default: return probe<0>(reps, iters);
  }
}
template <int OP>
static double probe(int reps, int iters) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * 65536) != cudaSuccess) return -1.0;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma_rate<OP><<<blocks, threads>>>(iters, 1.0, out);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dfma_rate<OP><<<blocks, threads>>>(iters, 1.0 + r, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess || ms <= 0) return -2.0;
  const double instr = (double)reps * blocks * threads * (double)iters * 8.0;
  return instr / (ms * 1e-3);
}

// Latency/ILP probe: one block of `warps` warps on one SM, each thread runs
// `chains` independent dependent-DFMA (or DMUL / DADD) chains; returns cycles
// per chain step measured with clock64 on warp 0.
namespace {
template <int CH, int OP>
__global__ void k_lat(int iters, double* out, long long* cyc) {
  double x[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) x[k] = 1.0 + threadIdx.x * 1e-9 + k;
  const double m = 0.9999999999, c = 1e-12;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (OP == 0) x[k] = __fma_rn(x[k], m, c);
      if (OP == 1) x[k] = __dmul_rn(x[k], m);
      if (OP == 2) x[k] = __dadd_rn(x[k], c);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int CH, int OP>
double lat_run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, 64);
  const int iters = 4096;
  k_lat<CH, OP><<<1, warps * 32>>>(iters, out, cyc);
  k_lat<CH, OP><<<1, warps * 32>>>(iters, out, cyc);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  cudaFree(out);
  cudaFree(cyc);
  return (double)h / iters;
}
}  // namespace
// cycles per iteration (each iteration = `chains` FP64 ops per thread)
extern "C" double eig33_probe_fp64_latency(int op, int chains, int warps) {
  if (op == 0) {
    if (chains == 1) return lat_run<1, 0>(warps);
    if (chains == 2) return lat_run<2, 0>(warps);
    if (chains == 4) return lat_run<4, 0>(warps);
    return lat_run<8, 0>(warps);
  }
  if (op == 1) return chains == 1 ? lat_run<1, 1>(warps) : lat_run<4, 1>(warps);
  return chains == 1 ? lat_run<1, 2>(warps) : lat_run<4, 2>(warps);
}

// Sustained FP64 rate on data that keeps every datapath bit toggling: eight
// independent chains of the chaotic map x <- x*x - 1.9999 (one DFMA each,
// bounded in [-2, 2]).  Run for seconds this is the FP64 roof of a long,
// power-capped step; a short run gives the burst rate.
namespace {
__global__ void __launch_bounds__(256) k_dfma_chaos(int iters, double* out) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = -1.5 + 3.0 * ((tid * 2654435761u + k * 40503u) & 0xFFFFu) / 65536.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], x[k], -1.9999);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}
}  // namespace

// DFMA thread-instructions per second over `seconds` of back-to-back launches.
extern "C" double eig33_probe_fp64_chaos(double seconds) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, 64) != cudaSuccess) return -1.0;
  const int blocks = sms * 8, threads = 256, iters = 8192;
  k_dfma_chaos<<<blocks, threads>>>(iters, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  int reps = 0;
  cudaEventRecord(e0);
  while (ms < seconds * 1e3f) {
    for (int r = 0; r < 8; ++r) k_dfma_chaos<<<blocks, threads>>>(iters, out);
    reps += 8;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess || ms <= 0) return -2.0;
  return (double)reps * blocks * threads * (double)iters * 8.0 / (ms * 1e-3);
}

// Pure stream with the kernel's traffic mix (72 B read, 24 B written per
// record), no FP64: out[i] = a[3i] ^ a[3i+1] ^ a[3i+2] on the bit patterns.
// Each warp load/store instruction covers 768 contiguous bytes.
namespace {
__global__ void __launch_bounds__(256) k_stream(const long long* __restrict__ a, long long n3,
                                                long long* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n3; i += stride)
    out[i] = __ldcs(a + 3 * i) ^ __ldcs(a + 3 * i + 1) ^ __ldcs(a + 3 * i + 2);
}
}  // namespace

extern "C" int eig33_probe_stream(const double* a, long long n, double* lam, void* stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_stream<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const long long*>(a), n * 3,
                                                       reinterpret_cast<long long*>(lam));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Data-path probe: k_fused's own TMA ring, tier tests and lambda stores with
// the steady-state arithmetic removed (the MEMONLY instantiation, which exists
// only in this measurement library, never in _eig33cuda.so), over a 16-B
// aligned batch.  bench.py's optional energy-model leg times it.
// ---------------------------------------------------------------------------
#define EIG33_TABLE_DECL static __device__ __align__(16)
#include "../../paper_2511_00292_b200/csrc/eig33_tables.h"
#include "../../paper_2511_00292_b200/csrc/eig33_fused.cuh"

extern "C" int eig33_probe_memonly(const double* d_a, size_t n, double* d_lam, void* stream) {
  using namespace eig33b;
  if (n == 0) return 0;
  if (!d_a || !d_lam || ((uintptr_t)d_a & 15u)) return 2;
  auto kern = k_fused<kEig, true, false, false, true>;
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // per call (and so per device): the attribute is per-device state
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)) !=
      cudaSuccess)
    return 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, sizeof(Smem)) != cudaSuccess ||
      occ < 1)
    return 1;
  const long long nchunks = (long long)((n + kChunk - 1) / kChunk);
  const long long nblk = (nchunks + kWarps - 1) / kWarps;
  const long long cap = (long long)sms * occ;
  kern<<<(unsigned)(nblk < cap ? nblk : cap), kThreads, sizeof(Smem), (cudaStream_t)stream>>>(
      d_a, (long long)n, nullptr, d_lam, nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
