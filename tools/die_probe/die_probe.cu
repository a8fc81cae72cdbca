// die_probe.cu -- research probe (not product): does reading memory homed on the
// SM's own die cost less energy than reading across the die-to-die link?
//   1. sm_lat: every SM times L2-hit loads to M granules -> SM/die clustering
//   2. granule_lat: SMs of one die time one L2-hit load per 2 KB granule of a
//      buffer -> near/far map of the buffer for that die
//   3. stream_sel: persistent read-only stream where each warp takes 2 KB
//      granules from a per-die work list (near, far or mixed assignment)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o tools/die_probe/libdie_probe.so tools/die_probe/die_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ long long clock_now() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : : "memory");
  return t;
}
// clock read that cannot issue before `dep` is available
__device__ __forceinline__ long long clock_after(unsigned long long dep) {
  long long t;
  asm volatile("{\n\t.reg .u64 d;\n\tmov.u64 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(t) : "l"(dep) : "memory");
  return t;
}
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// word 0 of every granule points at itself (for dependent-load chains)
__global__ void k_init_self(unsigned long long* buf, long long ngran, int gran_words) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < ngran;
       g += (long long)gridDim.x * blockDim.x)
    buf[g * gran_words] = (unsigned long long)(buf + g * gran_words);
}

// Average latency of 8 chained L2-hit loads of one word (after a warming load).
__device__ __forceinline__ int chain_lat(const unsigned long long* p, unsigned long long& sink) {
  p = (const unsigned long long*)ld_cg(p);  // warm
  const long long t0 = clock_now();
  // the chain's first address depends on t0 (t0 >> 63 is 0 at run time, but not
  // known to the compiler), so the clock read cannot sink below the loads
  p = (const unsigned long long*)((unsigned long long)p + (unsigned long long)(t0 >> 63));
#pragma unroll
  for (int r = 0; r < 8; ++r) p = (const unsigned long long*)ld_cg(p);
  if (p == nullptr) __trap();  // a branch on the last load: the clock read waits for it
  const long long t1 = clock_now();
  sink += (unsigned long long)p;
  return (int)((t1 - t0) / 8);
}

// grid: many blocks of 32 threads; lane 0 of each times M granules
__global__ void k_sm_lat(const unsigned long long* buf, int m, int stride_words, int reps,
                         int* sm_out, int* lat_out) {
  if (threadIdx.x != 0) return;
  const uint32_t s = smid();
  sm_out[blockIdx.x] = (int)s;
  unsigned long long sink = 0;
  for (int j = 0; j < m; ++j) {
    int best = 1 << 30;
    for (int r = 0; r < reps; ++r) {
      const int d = chain_lat(buf + (size_t)j * stride_words, sink);
      best = d < best ? d : best;
    }
    lat_out[blockIdx.x * m + j] = best;
  }
  if (sink == 0x123456789ull) lat_out[0] = -1;
}

// warps on SMs in `sm_mask` take granules from a shared counter and time them
__global__ void k_granule_lat(const unsigned long long* buf, long long ngran, int gran_words,
                              const uint32_t* sm_mask, int* lat_out, unsigned long long* done) {
  const uint32_t s = smid();
  if (!((sm_mask[s >> 5] >> (s & 31)) & 1u)) return;
  const int lane = threadIdx.x & 31;
  unsigned long long sink = 0;
  for (;;) {
    long long g = 0;
    if (lane == 0) g = (long long)atomicAdd(done, 1ull);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= ngran) break;
    if (lane == 0) lat_out[g] = chain_lat(buf + g * gran_words, sink);
  }
  if (sink == 0x123456789ull) lat_out[0] = -1;
}

// Persistent read-only stream: warps of an SM on die d take granules from
// list[d] (counter ctr[d]); each lane reads 64 B of the 2 KB granule.
__global__ void __launch_bounds__(256) k_stream_sel(const uint4* __restrict__ buf, int gran_u4,
                                                    const int* __restrict__ die_of_sm,
                                                    const long long* __restrict__ list0,
                                                    const long long* __restrict__ list1,
                                                    long long n0, long long n1,
                                                    unsigned long long* ctr, uint4* out) {
  const int d = die_of_sm[smid()];
  const long long* list = d ? list1 : list0;
  const long long nl = d ? n1 : n0;
  const int lane = threadIdx.x & 31;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (;;) {
    long long i = 0;
    if (lane == 0) i = (long long)atomicAdd(&ctr[d], 4ull);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= nl) break;
    uint4 v[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long gi = list[min(i + k, nl - 1)];
      const uint4* g = buf + gi * gran_u4;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[4 * k + q] = __ldcs(g + lane + 32 * q);  // 16 loads in flight
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      acc.x ^= v[k].x; acc.y ^= v[k].y; acc.z ^= v[k].z; acc.w ^= v[k].w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) out[0] = acc;
}

extern "C" {
int dp_init_self(void* buf, long long ngran, int gran_words) {
  k_init_self<<<1184, 256>>>((unsigned long long*)buf, ngran, gran_words);
  return cudaDeviceSynchronize();
}
int dp_sm_lat(const void* buf, int blocks, int m, int stride_words, int reps, int* sm_out, int* lat_out) {
  k_sm_lat<<<blocks, 32>>>((const unsigned long long*)buf, m, stride_words, reps, sm_out, lat_out);
  return cudaDeviceSynchronize();
}
int dp_granule_lat(const void* buf, long long ngran, int gran_words, const uint32_t* sm_mask,
                   int* lat_out, unsigned long long* done, int blocks) {
  k_granule_lat<<<blocks, 32>>>((const unsigned long long*)buf, ngran, gran_words, sm_mask, lat_out, done);
  return cudaDeviceSynchronize();
}
int dp_stream_sel(const void* buf, int gran_bytes, const int* die_of_sm, const long long* l0,
                  const long long* l1, long long n0, long long n1, unsigned long long* ctr,
                  void* out, int blocks, void* stream) {
  k_stream_sel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4*)buf, gran_bytes / 16, die_of_sm,
                                                          l0, l1, n0, n1, ctr, (uint4*)out);
  return (int)cudaGetLastError();
}
}
