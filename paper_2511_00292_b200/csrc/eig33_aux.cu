// eig33_aux.cu -- batched accuracy-study entry points:
// the naive / tensor invariant variants, eigvals_naive, and the invariant
// Jacobians.  They run on the hot path's staging and scheduling (eig33_fused.cuh):
// one 512-thread block per SM, per-warp TMA rings of 64-record chunks taken from
// a block-level counter, records read conflict-free from SMEM -- with a plain
// per-record body (no pipelining or tiers: the checked reference-order forms).
// Bit-exact against the reference like the hot path (compiled with --fmad=false).
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#define EIG33_TABLE_DECL static __device__ __align__(16)  // as in eig33_kernels.cu
#include "eig33_tables.h"
#include "eig33_fused.cuh"
#include "eig33_internal.h"

namespace eig33b {
namespace aux {

// invariants(a, Naive / NaiveTensor) (src/invariants.cpp:76-98)
struct InvVariantOp {
  int variant;
  double* inv;
  static constexpr bool kTables = false;
  void shift(size_t lo) { inv += lo * 4; }
  __device__ void operator()(const double m[9], long long r, const double*) const {
    store_inv(inv, r, invariants_variant(m, variant), ((uintptr_t)inv & 31u) == 0);
  }
};

// eigvals_naive (src/eigensolver.cpp:119-123): from_invariants on naive j2/j3,
// disc_naive, including the advisory (:54, tolerance from the stable kernels).
struct EigNaiveOp {
  double* lam;
  uint8_t* flags;
  static constexpr bool kTables = true;
  void shift(size_t lo) {
    lam += lo * 3;
    if (flags) flags += lo;
  }
  __device__ void operator()(const double m[9], long long r, const double* tab) const {
    const Inv v = invariants_variant(m, 1);
    const Lam L = from_invariants(m, v, tab);
    lam[r * 3 + 0] = L.l1;
    lam[r * 3 + 1] = L.l2;
    lam[r * 3 + 2] = L.l3;
    if (flags) {
      bool adv = false;
      if (v.disc < 0.0) {
        const Inv st = invariants_dag(m);
        adv = v.disc < -disc_tolerance(m, st.j2, st.j3);
      }
      flags[r] = adv ? EIG33_FLAG_ADVISORY : 0;
    }
  }
};

// jacobian_j2 / jacobian_j3 / jacobian_disc (src/invariants.cpp:60-74)
struct JacobiansOp {
  double *jj2, *jj3, *jdisc;
  static constexpr bool kTables = false;
  void shift(size_t lo) {
    if (jj2) jj2 += lo * 9;
    if (jj3) jj3 += lo * 9;
    if (jdisc) jdisc += lo * 9;
  }
  __device__ void operator()(const double m[9], long long r, const double*) const {
    double g[9];
    if (jj2) {
      jacobian_j2(m, g);
#pragma unroll
      for (int k = 0; k < 9; ++k) jj2[r * 9 + k] = g[k];
    }
    if (jj3) {
      jacobian_j3(m, g);
#pragma unroll
      for (int k = 0; k < 9; ++k) jj3[r * 9 + k] = g[k];
    }
    if (jdisc) {
      const Inv st = invariants_dag(m);
      jacobian_disc(m, st.j2, st.j3, g);
#pragma unroll
      for (int k = 0; k < 9; ++k) jdisc[r * 9 + k] = g[k];
    }
  }
};

// One record per lane per step, records staged through the warp's TMA ring.
template <class Op, bool TMA>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_map(const double* __restrict__ a, long long n, Op op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpRing R = make_ring(S, a, n, warp, lane);
  if (TMA && lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&R.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  sched_init(S);
  if (Op::kTables) copy_table(S.tab, eig33_tab);
  __syncthreads();
  ring_prologue<TMA>(R);
  for (uint32_t it = 0;; ++it) {
    int cnt;
    long long c, base;
    double* buf = ring_acquire<TMA>(R, it, c, base, cnt);
    if (!buf) break;
    if (it == 0) ring_kick<TMA>(R);
#pragma unroll
    for (int h = 0; h < kRPL; ++h) {
      if (32 * h >= cnt) {
        if (h == kRPL - 1) ring_release<TMA>(R, c, it, buf);
        continue;
      }
      double m[9];
      bool mod;
      ring_read(buf, lane, h, m, mod);
      if (h == kRPL - 1) ring_release<TMA>(R, c, it, buf);
      if (32 * h + lane < cnt) op(m, base + 32 * h + lane, S.tab);
    }
  }
}

template <class Op, bool TMA>
int launch_map_t(const double* a, size_t n, const Op& op, cudaStream_t st, const char* what) {
  auto kern = k_map<Op, TMA>;
  const size_t smem = sizeof(Smem);
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // the attribute is per-device state: set it on every call (cheap)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return EIG33_ECUDA;
  }
  const long long nchunks = (long long)((n + kChunk - 1) / kChunk);
  const long long nblk = (nchunks + kWarps - 1) / kWarps;
  const long long cap = (long long)sms * (occ > 0 ? occ : 1);
  kern<<<(unsigned)(nblk < cap ? nblk : cap), kThreads, smem, st>>>(a, (long long)n, op);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return EIG33_ECUDA;
  }
  return EIG33_OK;
}

template <class Op>
int launch_map(const double* a, size_t n, const Op& op, cudaStream_t st, const char* what) {
  // launches cover <= 2^31 records (32-bit chunk bookkeeping), as in eig33_kernels.cu
  constexpr size_t kMaxLaunch = size_t(1) << 31;
  for (size_t lo = 0; lo < n; lo += kMaxLaunch) {
    const size_t m = n - lo < kMaxLaunch ? n - lo : kMaxLaunch;
    Op piece = op;
    piece.shift(lo);
    const double* ap = a + lo * 9;
    const int rc = ((uintptr_t)ap & 15u) == 0 ? launch_map_t<Op, true>(ap, m, piece, st, what)
                                              : launch_map_t<Op, false>(ap, m, piece, st, what);
    if (rc) return rc;
  }
  return EIG33_OK;
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
  return aux::launch_map(d_a, n, aux::InvVariantOp{variant, d_inv}, (cudaStream_t)stream,
                         "k_map<invariants_variant> launch");
}

int eig33cu_eigvals_naive(const double* d_a, size_t n, double* d_lam, uint8_t* d_flags,
                          void* stream) {
  set_error("");
  if (n == 0) return EIG33_OK;
  if (!d_a || !d_lam) {
    set_error("eig33cu_eigvals_naive: null pointer");
    return EIG33_EINVAL;
  }
  return aux::launch_map(d_a, n, aux::EigNaiveOp{d_lam, d_flags}, (cudaStream_t)stream,
                         "k_map<eigvals_naive> launch");
}

int eig33cu_jacobians(const double* d_a, size_t n, double* d_jj2, double* d_jj3, double* d_jdisc,
                      void* stream) {
  set_error("");
  if (n == 0) return EIG33_OK;
  if (!d_a || (!d_jj2 && !d_jj3 && !d_jdisc)) {
    set_error("eig33cu_jacobians: bad argument");
    return EIG33_EINVAL;
  }
  return aux::launch_map(d_a, n, aux::JacobiansOp{d_jj2, d_jj3, d_jdisc}, (cudaStream_t)stream,
                         "k_map<jacobians> launch");
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
