// eig33_bench.cpp -- native C++ driver of the C ABI (no Python): generates a
// BASELINE config on the device, times eig33cu_eigvals with CUDA events, runs
// the host-buffer entry point end to end, and prints one line per measurement.
//
//   g++ -O2 -std=c++17 -I include tools/native/eig33_bench.cpp \
//       paper_2511_00292_b200/_eig33cuda.so -Wl,-rpath,$PWD/paper_2511_00292_b200 \
//       -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -o /tmp/eig33_bench
//   /tmp/eig33_bench [config=3] [log2 n=26] [launches=20]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "eig33_cuda.h"

#define CK(x)                                                                 \
  do {                                                                        \
    const int rc_ = (x);                                                      \
    if (rc_) {                                                                \
      std::fprintf(stderr, "%s -> %d: %s\n", #x, rc_, eig33cu_last_error()); \
      return 1;                                                               \
    }                                                                         \
  } while (0)
#define CU(x)                                                                             \
  do {                                                                                    \
    const cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                              \
      std::fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                    \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

int main(int argc, char** argv) {
  const int config = argc > 1 ? std::atoi(argv[1]) : 3;
  const int lg = argc > 2 ? std::atoi(argv[2]) : 26;
  const int launches = argc > 3 ? std::atoi(argv[3]) : 20;
  const size_t n = size_t(1) << lg;
  double *a = nullptr, *lam = nullptr;
  CU(cudaMalloc(&a, n * 9 * sizeof(double)));
  CU(cudaMalloc(&lam, n * 3 * sizeof(double)));
  CK(eig33cu_generate(config, 0x2511, 0, n, a, nullptr));
  for (int i = 0; i < 3; ++i) CK(eig33cu_eigvals(a, n, nullptr, lam, nullptr, nullptr));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  CU(cudaEventRecord(e0));
  for (int i = 0; i < launches; ++i) CK(eig33cu_eigvals(a, n, nullptr, lam, nullptr, nullptr));
  CU(cudaEventRecord(e1));
  CU(cudaEventSynchronize(e1));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  std::printf("device  config %d  n 2^%d  %.3f ms/launch  %.2f G records/s\n", config, lg,
              ms / launches, n * (double)launches / (ms * 1e-3) / 1e9);

  // end to end through the host-buffer entry point (pinned host memory)
  double *h_a = nullptr, *h_l = nullptr;
  CU(cudaMallocHost(&h_a, n * 9 * sizeof(double)));
  CU(cudaMallocHost(&h_l, n * 3 * sizeof(double)));
  CU(cudaMemcpy(h_a, a, n * 9 * sizeof(double), cudaMemcpyDeviceToHost));
  CK(eig33_eigvals_host(h_a, n, nullptr, h_l, nullptr, 0));
  const auto t0 = std::chrono::steady_clock::now();
  CK(eig33_eigvals_host(h_a, n, nullptr, h_l, nullptr, 0));
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("e2e     config %d  n 2^%d  %.3f s  %.3f G records/s  (H2D %.1f GB/s)\n", config, lg, s,
              n / s / 1e9, n * 72.0 / s / 1e9);
  std::vector<double> check(3);
  CU(cudaMemcpy(check.data(), lam, 24, cudaMemcpyDeviceToHost));
  const bool same = check[0] == h_l[0] && check[1] == h_l[1] && check[2] == h_l[2];
  std::printf("device and host paths agree on record 0: %s\n", same ? "yes" : "NO");
  cudaFreeHost(h_a);
  cudaFreeHost(h_l);
  cudaFree(a);
  cudaFree(lam);
  return same ? 0 : 1;
}
