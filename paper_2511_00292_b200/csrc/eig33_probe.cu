// eig33_probe.cu -- measurement helper for bench.py (not part of the C ABI
// contract): the achievable FP64-pipe issue rate of this GPU, used as the
// roofline denominator for the FP64-bound fused kernel.  MEASURED_PEAKS.json
// carries only HBM and bf16 peaks, so bench.py measures this on the box.
//
// Every thread runs 8 independent DFMA chains (enough ILP to cover the DFMA
// latency with 8 warps per SMSP); the result is written so nothing is dead.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__global__ void __launch_bounds__(256) k_dfma_rate(int iters, double seed, double* out) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = seed + (threadIdx.x + k) * 1e-9;
  const double m = 0.9999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[blockIdx.x] = s;  // practically never taken; defeats DCE
}
}  // namespace

// Returns DFMA warp-instructions*32 (thread-level FP64 instructions) per
// second measured over `reps` launches, or a negative value on error.
extern "C" double eig33_probe_fp64_rate(int reps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * 65536) != cudaSuccess) return -1.0;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma_rate<<<blocks, threads>>>(iters, 1.0, out);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dfma_rate<<<blocks, threads>>>(iters, 1.0 + r, out);
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
