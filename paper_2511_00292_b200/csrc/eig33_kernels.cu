// eig33_kernels.cu -- sm_100a kernels and device-pointer C ABI of the batched
// eig33 hot path (see include/eig33_cuda.h and DESIGN.md section 3).
//
// MUST be compiled with --fmad=false: the invariant arithmetic is bit-exact
// against the reference only without contraction (proj/src/CMakeLists.txt:9-10).
//
// Kernel map (device code in eig33_fused.cuh)
//   k_fused<MODE,TMA,INV,FLAGS>  persistent eigvals / eigvalss kernel: one
//       512-thread block per SM whose warps take 64-record chunks from a
//       block-level counter.  Each warp owns a 2-deep SMEM ring that lane 0
//       fills with cp.async.bulk (TMA 1D) on per-warp mbarriers -- no block
//       barrier in the loop.  The record loop is software-pipelined: one step =
//       eigenvalue stage of the previous record + invariants of the next, in one
//       block; the tier (steady / moderate / general, all inlined) is chosen per
//       warp.  With flags, the records with disc < 0 are queued per warp and
//       their non_real_advisory evaluated 32 at a time (advisory_flush).
//       Launched with programmatic dependent launch; outputs stored straight
//       from registers (invariants as one 256-bit store per record).
//   k_invariants<TMA>            invariants only, same ring and scheduler.
//   k_triple_angle               batched triple_angle.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <mutex>
#include <string>

// The table lives in global memory, not __constant__: the per-block copy into
// SMEM reads 32 different addresses per warp instruction, which the constant
// cache would serialise; from global they are coalesced 16-B loads (L2 hits
// after the first block).  See copy_table() in eig33_math.cuh.
#define EIG33_TABLE_DECL static __device__ __align__(16)
#include "eig33_tables.h"
#include "eig33_fused.cuh"
#include "eig33_internal.h"

namespace eig33b {

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

static int fail(int code, const char* what, cudaError_t e = cudaSuccess) {
  g_err = what;
  if (e != cudaSuccess) {
    g_err += ": ";
    g_err += cudaGetErrorString(e);
  }
  return code;
}

// Per-device launch geometry, computed once per kernel instantiation.  Host
// threads may launch concurrently (the multi-GPU driver runs one per device),
// so the first-use initialisation is serialised; the values are read back
// through atomics afterwards.
struct DevInfo {
  std::atomic<int> sms{0};
  std::atomic<int> occ[3][2][2][2] = {};
};
static DevInfo g_dev[64];
static std::mutex g_dev_mu;

template <int MODE, bool TMA, bool WI, bool WF>
static int launch_fused(const double* a, size_t n, double* inv, double* lam, uint8_t* flags,
                        cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaGetDevice", e);
  if (dev < 0 || dev >= 64) return fail(EIG33_EINVAL, "device index out of range");
  DevInfo& d = g_dev[dev];
  // eigvals with flags also carries the per-warp advisory queues
  const size_t smem = sizeof(Smem) + (MODE == kEig && WF ? (EIG33_ADVQ_SMEM ? sizeof(AdvRec) * kAdvR
                                                                           : sizeof(AdvEntry) * kAdvQ) *
                                                                kWarps
                                                          : 0);
  using KernFn = void (*)(const double*, long long, double*, double*, uint8_t*);
  KernFn kern;
  if constexpr (MODE == kInv)
    kern = k_invariants<TMA>;  // (no k_fused<kInv, ...> instantiation)
  else
    kern = k_fused<MODE, TMA, WI, WF>;
  std::atomic<int>& occ_slot = d.occ[MODE][TMA][WI][WF];
  int occ = occ_slot.load(std::memory_order_acquire);
  if (!occ) {
    std::lock_guard<std::mutex> lock(g_dev_mu);
    occ = occ_slot.load(std::memory_order_relaxed);
    if (!occ) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaFuncSetAttribute", e);
      int o = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, smem);
      if (e != cudaSuccess) return fail(EIG33_ECUDA, "occupancy query", e);
      if (!d.sms.load()) {
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return fail(EIG33_ECUDA, "SM count", e);
        d.sms.store(sms);
      }
      occ = o > 0 ? o : 1;
      occ_slot.store(occ, std::memory_order_release);
    }
  }
  const long long nchunks = (long long)((n + kChunk - 1) / kChunk);
  const long long nblk = (nchunks + kWarps - 1) / kWarps;  // at least one chunk per warp
  const long long cap = (long long)d.sms.load() * occ;
  const long long grid = nblk < cap ? nblk : cap;
#if EIG33_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a, (long long)n, inv, lam, flags);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "k_fused launch", e);
#else
  kern<<<(unsigned)grid, kThreads, smem, st>>>(a, (long long)n, inv, lam, flags);
#endif
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "k_fused launch", e);
  return EIG33_OK;
}

template <int MODE, bool TMA>
static int dispatch_out(const double* a, size_t n, double* inv, double* lam, uint8_t* flags,
                        cudaStream_t st) {
  if (inv) {
    return flags ? launch_fused<MODE, TMA, true, true>(a, n, inv, lam, flags, st)
                 : launch_fused<MODE, TMA, true, false>(a, n, inv, lam, flags, st);
  }
  return flags ? launch_fused<MODE, TMA, false, true>(a, n, inv, lam, flags, st)
               : launch_fused<MODE, TMA, false, false>(a, n, inv, lam, flags, st);
}

// Launches cover at most 2^31 records (32-bit chunk bookkeeping inside the
// kernel); larger batches -- beyond 154 GB of input, so only on future parts --
// are cut into such pieces (each 16-B aligned if the batch is).
template <int MODE>
static int dispatch(const double* a, size_t n, double* inv, double* lam, uint8_t* flags,
                    cudaStream_t st) {
  constexpr size_t kMaxLaunch = size_t(1) << 31;
  for (size_t lo = 0; lo < n; lo += kMaxLaunch) {
    const size_t m = n - lo < kMaxLaunch ? n - lo : kMaxLaunch;
    const double* ap = a + lo * 9;
    double* ip = inv ? inv + lo * 4 : nullptr;
    double* lp = lam ? lam + lo * 3 : nullptr;
    uint8_t* fp = flags ? flags + lo : nullptr;
    const bool aligned = ((uintptr_t)ap & 15u) == 0;
    const int rc = aligned ? dispatch_out<MODE, true>(ap, m, ip, lp, fp, st)
                           : dispatch_out<MODE, false>(ap, m, ip, lp, fp, st);
    if (rc) return rc;
  }
  return EIG33_OK;
}

}  // namespace eig33b

using namespace eig33b;

extern "C" {

int eig33cu_version(void) { return (1 << 16) | 0; }

#if EIG33_TIMELINE
// diagnostic builds only (tools/timeline.py): copy k_fused's per-warp timeline out
int eig33_debug_timeline(unsigned long long* out, int warps) {
  return cudaMemcpyFromSymbol(out, g_timeline, sizeof(unsigned long long) * 4 * (warps < 4096 ? warps : 4096)) ==
                 cudaSuccess
             ? 0
             : 1;
}
#endif
const char* eig33cu_last_error(void) { return g_err.c_str(); }

int eig33cu_invariants(const double* d_a, size_t n, double* d_inv, void* stream) {
  g_err.clear();
  if (n == 0) return EIG33_OK;
  if (!d_a || !d_inv) return fail(EIG33_EINVAL, "eig33cu_invariants: null pointer");
  return dispatch<kInv>(d_a, n, d_inv, nullptr, nullptr, (cudaStream_t)stream);
}

int eig33cu_eigvals(const double* d_a, size_t n, double* d_inv, double* d_lam, uint8_t* d_flags,
                    void* stream) {
  g_err.clear();
  if (n == 0) return EIG33_OK;
  if (!d_a || !d_lam) return fail(EIG33_EINVAL, "eig33cu_eigvals: null pointer");
  return dispatch<kEig>(d_a, n, d_inv, d_lam, d_flags, (cudaStream_t)stream);
}

int eig33cu_eigvalss(const double* d_a, size_t n, double* d_inv, double* d_lam, uint8_t* d_flags,
                     void* stream) {
  g_err.clear();
  if (n == 0) return EIG33_OK;
  if (!d_a || !d_lam) return fail(EIG33_EINVAL, "eig33cu_eigvalss: null pointer");
  return dispatch<kSym>(d_a, n, d_inv, d_lam, d_flags, (cudaStream_t)stream);
}

int eig33cu_triple_angle(const double* d_j3, const double* d_disc, size_t n, double* d_phi,
                         void* stream) {
  g_err.clear();
  if (n == 0) return EIG33_OK;
  if (!d_j3 || !d_disc || !d_phi) return fail(EIG33_EINVAL, "eig33cu_triple_angle: null pointer");
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = (long long)((n + kThreads - 1) / kThreads);
  const long long grid = blocks < 8LL * sms ? blocks : 8LL * sms;
  k_triple_angle<<<(unsigned)grid, kThreads, 0, (cudaStream_t)stream>>>(d_j3, d_disc, (long long)n,
                                                                       d_phi);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "k_triple_angle launch", e);
  return EIG33_OK;
}

}  // extern "C"
