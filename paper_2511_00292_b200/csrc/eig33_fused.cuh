// eig33_fused.cuh -- device code of the batched eig33 hot path: the
// persistent fused kernel k_fused, k_invariants, the deferred advisory and
// k_triple_angle.  Included by eig33_kernels.cu (the
// product: launch plumbing + device-pointer C ABI) and by the measurement
// probes under tools/probes (the only place k_fused's MEMONLY form is
// instantiated; the product library never contains it).
//
// MUST be compiled with --fmad=false: the invariant arithmetic is bit-exact
// against the reference only without contraction (proj/src/CMakeLists.txt:9-10).
// The includer defines EIG33_TABLE_DECL and includes eig33_tables.h first.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "eig33_math.cuh"
#include "../../include/eig33_cuda.h"

namespace eig33b {

#ifndef EIG33_PDL
#define EIG33_PDL 1
#endif
// One 512-thread block (16 warps) per SM: the 128-register budget allows 16
// warps per SM either way, and one block lets all 16 share one dynamic chunk
// counter (EIG33_DYN) -- measured +5.5% on config 3 and +14% on config 5
// against two 256-thread blocks per SM (tools/variant_compare.py).
#ifndef EIG33_THREADS
#define EIG33_THREADS 512
#endif
constexpr int kThreads = EIG33_THREADS;  // threads per block
constexpr int kWarps = kThreads / 32;
#ifndef EIG33_RPL
#define EIG33_RPL 2
#endif
constexpr int kRPL = EIG33_RPL;  // records per lane per chunk (1, 2 or 4)
static_assert(kRPL == 1 || kRPL == 2 || kRPL == 4, "kRPL must be 1, 2 or 4");
constexpr int kChunk = 32 * kRPL;  // records per warp chunk
#ifndef EIG33_STAGES
#define EIG33_STAGES (4 / EIG33_RPL)
#endif
constexpr int kStages = EIG33_STAGES;  // per-warp TMA ring depth (power of two)
static_assert((kStages & (kStages - 1)) == 0, "kStages must be a power of two");
#ifndef EIG33_MIN_BLOCKS
#define EIG33_MIN_BLOCKS 1
#endif
constexpr int kMinBlocks = EIG33_MIN_BLOCKS;  // resident blocks per SM the register budget targets
constexpr int kTabDoubles = EIG33_TAB_N;
constexpr uint32_t kChunkBytes = kChunk * 9 * sizeof(double);  // 2304 * kRPL
constexpr uint8_t kPending = 0x4;  // internal: advisory still to be evaluated

enum Mode { kEig = 0, kInv = 1, kSym = 2 };

struct __align__(16) Smem {
  double in[kWarps][kStages][kChunk * 9];
  double tab[kTabDoubles + 7];
  unsigned long long bar[kWarps][kStages];
  int next;  // block-level chunk counter (EIG33_DYN)
};

// In-kernel advisory queue (eigvals with flags).  The advisory
// (src/eigensolver.cpp:54) needs disc_tolerance -- the Jacobian of disc and two
// Frobenius norms, ~110 FP64 operations -- only for records with disc < 0 (0%
// of configs 1-3, 37% of config 4).  Evaluating it in every step would cost
// every lane of a warp whenever one lane is pending; instead each warp queues
// its pending records (index + j2, j3, disc) in a 64-entry SMEM ring and
// evaluates them 32 at a time, one per lane, re-reading the 72-B record from
// global memory -- an L2 hit: the warp's TMA brought it on chip moments ago.
// (The previous design, a deferred kernel re-reading every pending record
// from HBM, cost 72 us next to k_fused's 121 us on config 4.  Flushing 64 at a
// time, two records per lane from a 96-entry queue, measured slower: 23.3 vs
// 24.7 G records/s on config 4.)
// EIG33_FLUSH_PROBE (measurement builds only): 1 = never flush (pending flag
// bytes stay unwritten), 2 = flush loads the records but skips the arithmetic.
// On config 4 with invariants and flags (tools/store_mix.py, 2^22 records):
// lambda alone 24.5 ps/record, + pushes and stores without any flush 26.3,
// + the flush's loads and flag stores 29.0, + the arithmetic 31.8.  Staging
// the records into SMEM ahead of the flush with cp.async (one step early, so
// the L2 round trip is off the flushing warp's path) measured slower: 29.6 vs
// 31.0 G records/s on config 4, and -1.8% on config 3 with invariants (the
// 225-KB SMEM carve-out leaves L1 almost nothing); not adopted.
#ifndef EIG33_FLUSH_PROBE
#define EIG33_FLUSH_PROBE 0
#endif
struct AdvEntry {
  long long idx;
  double j2, j3, disc;
};
constexpr uint32_t kAdvQ = 64;        // entries per warp: >= 2 x 32
constexpr uint32_t kAdvFlushAt = 32;  // a flush evaluates 32, one per lane

// Evaluate `count` (<= 32) queued records starting at `head`, one per lane,
// and write their final flag bytes.  Out of line: its registers never enter
// the steady-state loop's allocation.
static __device__ __noinline__ void advisory_flush(const double* __restrict__ a, uint8_t* __restrict__ flags,
                                            const AdvEntry* q, uint32_t head, uint32_t count) {
  __syncwarp();  // queue entries were written by other lanes
  const uint32_t lane = threadIdx.x & 31u;
  if (lane < count) {
    const AdvEntry e = q[(head + lane) % kAdvQ];
    EIG33_CHECK(e.idx >= 0);
    double m[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) m[k] = __ldg(a + e.idx * 9 + k);
#if EIG33_FLUSH_PROBE == 2  // measurement: loads only
    flags[e.idx] = (m[0] + m[1] + m[2] + m[3] + m[4] + m[5] + m[6] + m[7] + m[8] + e.disc) < 0.0;
#else
    flags[e.idx] = advisory(m, Inv{0.0, e.j2, e.j3, e.disc}) ? EIG33_FLAG_ADVISORY : 0;
#endif
  }
  __syncwarp();  // the slots may be refilled by the next push
}

// EIG33_ADVQ_SMEM=1 (measurement variant): the queue holds the records
// themselves (copied from the SMEM ring at push time, 104 B per entry, 32
// entries per warp, flushed before it would overflow), so a flush reads no
// global memory at all.  The ring stage of a chunk is then handed back only
// after the chunk's last step.
#ifndef EIG33_ADVQ_SMEM
#define EIG33_ADVQ_SMEM 0
#endif
struct AdvRec {
  double m[9];
  double j2, j3, disc;
  long long idx;
};
constexpr uint32_t kAdvR = 32;
static __device__ __noinline__ void advisory_flush_smem(uint8_t* __restrict__ flags, const AdvRec* q,
                                                 uint32_t count) {
  __syncwarp();
  const uint32_t lane = threadIdx.x & 31u;
  if (lane < count) {
    const AdvRec& e = q[lane];
    double m[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) m[k] = e.m[k];
    flags[e.idx] = advisory(m, Inv{0.0, e.j2, e.j3, e.disc}) ? EIG33_FLAG_ADVISORY : 0;
  }
  __syncwarp();
}


__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

// Programmatic dependent launch: k_fused / k_invariants are launched with
// programmatic stream serialisation, so their blocks may start while the
// previous kernel on the stream drains.  Everything before pdl_wait() touches
// only SMEM (barrier init, table copy from a read-only global array); every
// read or write of caller buffers comes after it, and griddepcontrol.wait
// returns only once the previous grid has completed and its writes are
// visible.  pdl_trigger() lets the next kernel do the same.
__device__ __forceinline__ void pdl_trigger() {
#if EIG33_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if EIG33_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// EIG33_TIMELINE=1 (diagnostic build, tools/timeline.py): each warp of k_fused
// records %globaltimer at entry, after griddepcontrol.wait, when its first
// chunk has landed, and at exit.  Never in the product build.
#ifndef EIG33_TIMELINE
#define EIG33_TIMELINE 0
#endif
#if EIG33_TIMELINE
__device__ unsigned long long g_timeline[4096][4];
__device__ __forceinline__ void tl_mark(int slot) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (w < 4096) g_timeline[w][slot] = t;
  }
}
#else
__device__ __forceinline__ void tl_mark(int) {}
#endif

__device__ __forceinline__ void load_tables(double* tab) {
  copy_table(tab, eig33_tab);
}

struct Tabs {
  const double* tab;
};

// The checked reference-order kernels return the same bits as the moderate
// ones on moderate records, so a warp with any non-moderate lane runs the
// checked kernel on every lane rather than both kernels one after the other
// (divergent lanes would serialise them).  `mask`: the lanes executing the call.
__device__ __forceinline__ Inv invariants_warp(const double m[9], bool mod, unsigned mask) {
  // checked form: the always-valid CSE DAG (231 ops vs 341 in reference order)
  return __all_sync(mask, mod) ? invariants_moderate(m) : invariants_dag(m);
}

// Stage 1 of a record: symmetry gate (eigvalss), invariants, flag bits, and
// the eigen-stage carry.  Moderate records (every |a_ij| in [2^-100,2^100), the
// common case) use the CSE DAG; the rest the checked reference-order kernel.
// Both produce the reference's bits.
template <int MODE, bool WANT_FLAGS>
__device__ __forceinline__ void stage1(double m[9], bool& mod, Inv& v, Carry& c, uint8_t& f,
                                       bool& bad) {
  f = 0;
  bad = false;
  if (MODE == kSym) {
    if (not_symmetric(m)) {
      bad = true;
      mod = false;
      f = EIG33_FLAG_NOT_SYMMETRIC;
    }
    m[3] = m[1];  // mirror the upper triangle, src/eigensolver.cpp:108-111
    m[6] = m[2];
    m[7] = m[5];
  }
  v = invariants_warp(m, mod, 0xffffffffu);
  if (MODE == kSym && bad) {
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    v.i1 = v.j2 = v.j3 = v.disc = qnan;
  }
  if (MODE == kEig && WANT_FLAGS && v.disc < 0.0) f = kPending;
  c = Carry{v.i1, v.j2, v.j3, v.disc, m[0], m[4], m[8]};
}

// Stage 2 (eigenvalues) of a record from its carry, general form; called by
// whole warps.  As in invariants_warp, the general (any-input) form serves
// every lane once any lane needs it (same bits on moderate carries).
__device__ __forceinline__ Lam stage2(const Carry& c, bool mod, bool bad, const Tabs& T) {
  Lam L = __all_sync(0xffffffffu, mod || bad) ? eig_moderate_bl(c, T.tab) : eig_general_bl(c, T.tab);
  if (bad) {
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    L = Lam{qnan, qnan, qnan};
  }
  return L;
}

// Slow tiers of the record pipeline.  Both are inlined: the general tier used
// to be a real call (in reference order, with arrays, inlining it made ptxas
// spill inside the steady-state loop and cost 3x); as straight-line any-input
// forms it inlines with no spills and measured +20% on config 4 and +7% on
// config 5 with flags (tools/variant_compare.py; EIG33_GENERAL_INLINE=0 keeps
// the call).
#ifndef EIG33_GENERAL_INLINE
#define EIG33_GENERAL_INLINE 1
#endif

#if EIG33_GENERAL_INLINE
#define EIG33_GENERAL_ATTR __forceinline__
#else
#define EIG33_GENERAL_ATTR __noinline__
#endif
struct M9 {
  double e[9];
};
struct StepOut {
  Lam L;
  Inv v;
  uint8_t f;
  bool bad, mod;
};

// Tier B, warp-uniform: every lane moderate but some carried record has
// j2 <= 0 or disc <= 0: branch-free eig_moderate_bl interleaved with the DAG.
// Inlined: measured +6% on config 4 (every warp step here) and +1.3% on the
// sustained config-3 bench against an out-of-line call (argument moves, no
// overlap with the loads/stores around the call).
template <int MODE, bool WANT_FLAGS>
__device__ __forceinline__ StepOut tier_moderate(M9 mm, Carry pc, const double* tab) {
  StepOut o;
  o.L = eig_moderate_bl(pc, tab);
  o.v = invariants_moderate(mm.e);
  o.f = (MODE == kEig && WANT_FLAGS && o.v.disc < 0.0) ? kPending : 0;
  o.bad = false;
  o.mod = true;
  return o;
}

// Tier C, warp-uniform: some lane holds a record outside the moderate range
// (zeros mixed with tiny entries, subnormals, extreme exponents, inf/NaN) or an
// eigvalss reject.  Straight-line any-input forms for both stages -- the
// always-valid invariant DAG and eig_general_bl (selects, no per-lane special
// branches) -- so the scheduler interleaves them like the moderate tier.
template <int MODE, bool WANT_FLAGS>
__device__ EIG33_GENERAL_ATTR StepOut tier_general(M9 mm, bool sym_ok, bool mod, Carry pc, bool pbad,
                                                   const double* tab) {
  StepOut o;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  o.L = eig_general_bl(pc, tab);
  if (pbad) o.L = Lam{qnan, qnan, qnan};
  o.v = invariants_dag(mm.e);
  o.bad = MODE == kSym && !sym_ok;  // (already mirrored: the gate verdict decides)
  o.f = 0;
  if (o.bad) {
    o.v.i1 = o.v.j2 = o.v.j3 = o.v.disc = qnan;
    o.f = EIG33_FLAG_NOT_SYMMETRIC;
  }
  if (MODE == kEig && WANT_FLAGS && o.v.disc < 0.0) o.f = kPending;
  o.mod = mod && !o.bad;
  return o;
}

// One record's invariants {i1, j2, j3, disc}: a single 256-bit store
// (STG.256, sm_100) when the output is 32-B aligned -- a warp then writes
// 1 KB of whole sectors -- else four 8-B stores.
__device__ __forceinline__ void store_inv(double* __restrict__ inv, long long r, const Inv& v, bool a32) {
  double* p = inv + r * 4;
  if (a32) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.i1), "d"(v.j2), "d"(v.j3),
                 "d"(v.disc)
                 : "memory");
  } else {
    p[0] = v.i1;
    p[1] = v.j2;
    p[2] = v.j3;
    p[3] = v.disc;
  }
}

// Per-warp record pipeline.  Work unit = a chunk of kChunk consecutive
// records (kRPL per lane).  Lane 0 streams the warp's chunks HBM -> SMEM with
// cp.async.bulk into a kStages-deep per-warp ring completed on per-warp
// mbarriers: no block-wide barrier in the loop.
//
// Chunk assignment (EIG33_DYN=1, the default): block b owns the chunks
// b, b + G, b + 2G, ... (G = grid size) and its warps take them from a
// block-level SMEM counter -- each warp's first kStages chunks statically,
// every further one with one shared-memory atomicAdd when a ring stage is
// handed back to the TMA engine (kStages chunks ahead of use, so the atomic's
// latency is hidden).  The warp scheduler favours some warps over others
// (greedy-then-oldest); with a static split the favoured warps finish early
// and the SM runs its last microseconds with too few warps to hide the FP64
// latency.  Dynamic assignment keeps every warp busy to within one chunk of
// the block's end.  (EIG33_DYN=0: warp gw takes chunks gw, gw + W, ...)
#ifndef EIG33_DYN
#define EIG33_DYN 1
#endif
static_assert(kStages == 2, "the chunk bookkeeping below holds exactly two ring stages");
// Chunk geometry.  Chunk ids [0, n64 - ts) are 64-record chunks; the last ts
// full chunks are cut into 2*ts 32-record half-chunks (EIG33_SPLIT_TAIL chunks
// per warp of the grid: the block counter hands them out last, so a launch
// ends on half-size work units and its SMs finish closer together); a ragged
// remainder of n % 64 records is the last chunk (no TMA).  "full" counts the
// TMA-able chunks (64- or 32-record).
#ifndef EIG33_SPLIT_TAIL
#define EIG33_SPLIT_TAIL 0
#endif
struct WarpRing {
  double* ring;
  unsigned long long* bars;
  const double* a;
  long long n, nchunks, full, n64, ts;
  long long b, G, gw, W;  // block, grid size, global warp, total warps
  int* next;              // block counter in SMEM
  int warp, lane;
  long long cid0, cid1;   // chunk of ring stage 0 / 1 (lane 0's values are authoritative)
};
__device__ __forceinline__ WarpRing make_ring(Smem& S, const double* a, long long n, int warp, int lane) {
  WarpRing R;
  R.ring = S.in[warp][0];
  R.bars = S.bar[warp];
  R.a = a;
  R.n = n;
  R.n64 = n / kChunk;
  R.ts = 0;
  if (EIG33_SPLIT_TAIL > 0 && kRPL == 2) {
    const long long want = (long long)EIG33_SPLIT_TAIL * kWarps * gridDim.x;
    R.ts = want < R.n64 ? want : R.n64;
  }
  R.full = R.n64 + R.ts;
  R.nchunks = R.full + (n % kChunk ? 1 : 0);
  R.b = blockIdx.x;
  R.G = gridDim.x;
  R.gw = (long long)blockIdx.x * kWarps + warp;
  R.W = (long long)gridDim.x * kWarps;
  R.next = &S.next;
  R.warp = warp;
  R.lane = lane;
  R.cid0 = R.cid1 = 0;
  return R;
}
// first record and record count of chunk c (c < nchunks)
__device__ __forceinline__ long long chunk_start(const WarpRing& R, long long c) {
  const long long c64 = R.n64 - R.ts;
  if (c < c64) return c * kChunk;
  if (c < R.full) return c64 * kChunk + (c - c64) * 32;
  return R.n64 * kChunk;
}
__device__ __forceinline__ int chunk_cnt(const WarpRing& R, long long c) {
  if (c < R.n64 - R.ts) return kChunk;
  if (c < R.full) return 32;
  return (int)(R.n - R.n64 * kChunk);
}
// First chunk of ring stage s, and the chunk that follows c when its stage is
// refilled (lane 0 only).
__device__ __forceinline__ long long sched_first(const WarpRing& R, int s) {
  return EIG33_DYN ? R.b + (long long)(R.warp + s * kWarps) * R.G : R.gw + (long long)s * R.W;
}
__device__ __forceinline__ long long sched_next(const WarpRing& R, long long c) {
  return EIG33_DYN ? R.b + (long long)atomicAdd(R.next, 1) * R.G : c + (long long)kStages * R.W;
}
// thread 0, before the block barrier: the counter starts past the static chunks
__device__ __forceinline__ void sched_init(Smem& S) {
  if (threadIdx.x == 0) S.next = kStages * kWarps;
}

// EIG33_LAZY2=1 (default): at launch each warp asks only for its first chunk;
// the second ring stage is requested once the first has landed (ring_kick).
// Every warp of the grid requests its first bytes at the same moment, so
// halving that burst brings the first chunks in sooner (latest first chunk of
// a 2^18-record launch 4.1 -> 2.8 us after griddepcontrol.wait; +0.5-1% on
// configs 2-5, tools/variant_compare.py).
#ifndef EIG33_LAZY2
#define EIG33_LAZY2 1
#endif

template <bool TMA>
__device__ __forceinline__ void ring_issue(const WarpRing& R, int s) {
  const long long c = s ? R.cid1 : R.cid0;
  if (TMA && c < R.full) {
    const long long st = chunk_start(R, c);
    const uint32_t bytes = (uint32_t)chunk_cnt(R, c) * 72u;
    mbar_expect_tx(&R.bars[s], bytes);
    EIG33_CHECK(st + chunk_cnt(R, c) <= R.n);
    bulk_load(R.ring + s * (kChunk * 9), R.a + st * 9, bytes, &R.bars[s]);
  }
}
template <bool TMA>
__device__ __forceinline__ void ring_prologue(WarpRing& R) {
  if (R.lane == 0) {
    R.cid0 = sched_first(R, 0);
    R.cid1 = sched_first(R, 1);
    ring_issue<TMA>(R, 0);
    if (!EIG33_LAZY2) ring_issue<TMA>(R, 1);
  }
}
// the deferred second stage (EIG33_LAZY2), after the first chunk has landed
template <bool TMA>
__device__ __forceinline__ void ring_kick(const WarpRing& R) {
  if (EIG33_LAZY2 && R.lane == 0) ring_issue<TMA>(R, 1);
}

// Iteration it of this warp: the chunk in ring stage it % 2 (c, broadcast
// from lane 0; nullptr when the warp's work is done); waits for its TMA (or
// loads it cooperatively: misaligned input / ragged last chunk).
template <bool TMA>
__device__ __forceinline__ double* ring_acquire(const WarpRing& R, uint32_t it, long long& c, long long& base,
                                                int& cnt) {
  const uint32_t stage = it & (kStages - 1);
  c = __shfl_sync(0xffffffffu, stage ? R.cid1 : R.cid0, 0);
  if (c >= R.nchunks) return nullptr;
  double* buf = R.ring + stage * (kChunk * 9);
  base = chunk_start(R, c);
  cnt = chunk_cnt(R, c);
  if (TMA && c < R.full) {
    mbar_wait(&R.bars[stage], (it / kStages) & 1u);
  } else {
    const double* src = R.a + base * 9;
#pragma unroll
    for (int j = 0; j < 9 * kRPL; ++j) {
      const int e = R.lane + 32 * j;
      buf[e] = e < cnt * 9 ? __ldg(src + e) : 1.0;
    }
    __syncwarp();
  }
  return buf;
}
// Record h (0..kRPL-1) of this lane from the chunk buffer; `mod` consumes all
// nine loads, so once every record of the chunk is read the stage can be
// handed back to the TMA engine (ring_release).
__device__ __forceinline__ void ring_read(const double* buf, int lane, int h, double m[9],
                                          bool& mod) {
#pragma unroll
  for (int j = 0; j < 9; ++j) m[j] = buf[(lane + 32 * h) * 9 + j];
  mod = is_moderate(m);
  if (!mod) mod = is_moderate_or_zero(m);
}
template <bool TMA>
__device__ __forceinline__ void ring_release(WarpRing& R, long long c, uint32_t it, double* buf) {
  __syncwarp();
  if (R.lane == 0) {
    const uint32_t stage = it & (kStages - 1);
    const long long nc = sched_next(R, c);
    if (stage) R.cid1 = nc;
    else R.cid0 = nc;
    if (TMA && nc < R.full) {
      const long long st = chunk_start(R, nc);
      const uint32_t bytes = (uint32_t)chunk_cnt(R, nc) * 72u;
      mbar_expect_tx(&R.bars[stage], bytes);
      EIG33_CHECK(st + chunk_cnt(R, nc) <= R.n);
      bulk_load(buf, R.a + st * 9, bytes, &R.bars[stage]);
    }
  }
}

// Persistent fused kernel, software-pipelined across records: iteration i
// computes the invariants of chunk i and the eigenvalue stage of chunk i-1 in
// one basic block (both branch-free in the moderate case), so the long serial
// transcendental chain of one record overlaps the wide invariant DAG of the
// next.  Outputs go straight from registers to HBM (a warp's lambda stores
// cover one contiguous 768-B run; L2 merges the sectors).
// MEMONLY (measurement probe eig33_probe_memonly only): the same ring, tier
// tests and stores with the steady-state arithmetic removed -- the kernel's own
// data-movement energy for the energy roof in bench.py.
template <int MODE, bool TMA, bool WANT_INV, bool WANT_FLAGS, bool MEMONLY = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    k_fused(const double* __restrict__ a, long long n, double* __restrict__ inv,
            double* __restrict__ lam, uint8_t* __restrict__ flags) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpRing R = make_ring(S, a, n, warp, lane);
  const bool inv32 = ((uintptr_t)inv & 31u) == 0;

  if (TMA && lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&R.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  sched_init(S);
  tl_mark(0);
  pdl_trigger();
  load_tables(S.tab);
  __syncthreads();  // tables + barrier init + chunk counter; the only block-wide barrier
  pdl_wait();
  tl_mark(1);
  const Tabs T{S.tab};
  ring_prologue<TMA>(R);

  double m[9];
  bool mod, bad, pmod, pbad, pfast, pvalid;
  Inv v{};  // set by every stage1/step before store_stage1 reads it
  Carry pc;
  uint8_t f;
  long long pr;  // record index of the carried stage
  constexpr bool kQueue = MODE == kEig && WANT_FLAGS;
  AdvEntry* advq = kQueue ? reinterpret_cast<AdvEntry*>(smem_raw + sizeof(Smem)) + warp * kAdvQ : nullptr;
#if EIG33_ADVQ_SMEM
  AdvRec* advr = kQueue ? reinterpret_cast<AdvRec*>(smem_raw + sizeof(Smem)) + warp * kAdvR : nullptr;
#endif
  uint32_t qh = 0, qt = 0;  // queue head / tail (warp-uniform, monotone counts)
  // src: this lane's record in the ring (EIG33_ADVQ_SMEM copies it into the queue)
  auto store_stage1 = [&](long long r, bool valid, const double* src) {
    const bool pend = kQueue && valid && f == kPending;
    if (kQueue) {  // pending records go to the advisory queue, their flag byte comes later
      const unsigned pm = __ballot_sync(0xffffffffu, pend);
      if (pm) {
#if EIG33_ADVQ_SMEM
        if (qt + __popc(pm) > kAdvR) {
          advisory_flush_smem(flags, advr, qt);
          qt = 0;
        }
        if (pend) {
          AdvRec& e = advr[qt + __popc(pm & ((1u << lane) - 1u))];
#pragma unroll
          for (int k = 0; k < 9; ++k) e.m[k] = src[k];
          e.j2 = v.j2;
          e.j3 = v.j3;
          e.disc = v.disc;
          e.idx = r;
        }
        qt += __popc(pm);
#else
        (void)src;
        if (pend) {
          const uint32_t pos = (qt + __popc(pm & ((1u << lane) - 1u))) % kAdvQ;
          advq[pos] = AdvEntry{r, v.j2, v.j3, v.disc};
        }
        qt += __popc(pm);
        if (EIG33_FLUSH_PROBE != 1 && qt - qh >= kAdvFlushAt) {
          advisory_flush(a, flags, advq, qh, 32u);
          qh += 32u;
        }
#endif
      }
    }
    if (!valid) return;
    EIG33_CHECK(r >= 0 && r < R.n);
    if (WANT_INV) store_inv(inv, r, v, inv32);
    if (MODE != kInv && WANT_FLAGS && !pend) flags[r] = f;
  };
  auto store_lam = [&](const Lam& L) {
    if (!pvalid) return;
    EIG33_CHECK(pr >= 0 && pr < R.n);
    lam[pr * 3 + 0] = L.l1;
    lam[pr * 3 + 1] = L.l2;
    lam[pr * 3 + 2] = L.l3;
  };
  // One step of the record pipeline: stage 2 of the carried record, stage 1 of m.
  auto step = [&](long long r, bool valid, const double* src) {
    Carry nc;
    Lam L;
    bool sym_ok = true;
    if (MODE == kSym) {
      // eigvalss gate + mirror (src/eigensolver.cpp:98-111) ahead of the
      // steady-state test; mirroring keeps a moderate record moderate.
      sym_ok = !not_symmetric(m);
      m[3] = m[1];
      m[6] = m[2];
      m[7] = m[5];
    }
    // Warp-uniform tier choice, so a warp never runs two tiers for one step.
    if (__all_sync(0xffffffffu, sym_ok && mod && pfast)) {
      // steady state: one branch-free block (stage 2 of pr, stage 1 of r);
      // the long transcendental chain is written first so the scheduler
      // starts it early and fills its latency with the invariant DAG.
      if constexpr (MEMONLY) {  // measurement probe: same data movement, no arithmetic
        L = Lam{pc.a0, pc.a4, pc.a8};
        v = Inv{m[0], 1.0, m[1], 1.0};
      } else {
        L = eig_fast(pc, T.tab);
        v = invariants_moderate(m);
      }
      if (MODE == kEig && WANT_FLAGS) f = v.disc < 0.0 ? kPending : 0;
      if (MODE == kSym) f = 0;
      bad = false;
    } else {
      M9 mm;
#pragma unroll
      for (int k = 0; k < 9; ++k) mm.e[k] = m[k];
      StepOut o;
      if (__all_sync(0xffffffffu, sym_ok && mod && pmod))
        o = tier_moderate<MODE, WANT_FLAGS>(mm, pc, T.tab);
      else
        o = tier_general<MODE, WANT_FLAGS>(mm, sym_ok, mod, pc, pbad, T.tab);
      L = o.L;
      v = o.v;
      f = o.f;
      bad = o.bad;
      mod = o.mod;
    }
    nc = Carry{v.i1, v.j2, v.j3, v.disc, m[0], m[4], m[8]};
    store_lam(L);
    store_stage1(r, valid, src);
    pc = nc;
    pmod = mod;
    pfast = mod && fast_carry(v);
    pbad = bad;
    pr = r;
    pvalid = valid;
  };

  // ---- prologue: first chunk; stage 1 of its first record ----
  int cnt;
  long long c, base;
  double* buf = ring_acquire<TMA>(R, 0, c, base, cnt);
  if (!buf) return;  // no chunk for this warp (small batch)
  ring_kick<TMA>(R);
  tl_mark(2);
  // with the record-copying advisory queue the stage is handed back only
  // after the chunk's last step has read its pending records
  constexpr bool kLateRelease = kQueue && EIG33_ADVQ_SMEM;
  ring_read(buf, lane, 0, m, mod);
  if (kRPL == 1 && !kLateRelease) ring_release<TMA>(R, c, 0, buf);
  stage1<MODE, WANT_FLAGS>(m, mod, v, pc, f, pbad);
  pmod = mod;
  pfast = mod && fast_carry(v);
  pr = base + lane;
  pvalid = lane < cnt;
  store_stage1(pr, pvalid, buf + lane * 9);
  if (kRPL == 1 && kLateRelease) ring_release<TMA>(R, c, 0, buf);
  // Record slot h of the current chunk: one pipeline step; a slot past the
  // chunk's records (a 32-record half chunk) is skipped, warp-uniformly.
  auto slot = [&](int h, uint32_t it) {
    const bool last = h == kRPL - 1;
    if (32 * h >= cnt) {
      if (last) ring_release<TMA>(R, c, it, buf);
      return;
    }
    ring_read(buf, lane, h, m, mod);
    if (last && !kLateRelease) ring_release<TMA>(R, c, it, buf);
    step(base + 32 * h + lane, 32 * h + lane < cnt, buf + (lane + 32 * h) * 9);
    if (last && kLateRelease) ring_release<TMA>(R, c, it, buf);
  };
#pragma unroll
  for (int h = 1; h < kRPL; ++h) slot(h, 0);
  for (uint32_t it = 1;; ++it) {
    buf = ring_acquire<TMA>(R, it, c, base, cnt);
    if (!buf) break;
#pragma unroll
    for (int h = 0; h < kRPL; ++h) slot(h, it);
  }
  store_lam(stage2(pc, pmod, pbad, T));
#if EIG33_ADVQ_SMEM
  if (kQueue && qt) advisory_flush_smem(flags, advr, qt);
#else
  while (kQueue && EIG33_FLUSH_PROBE != 1 && qt != qh) {  // < kAdvFlushAt left
    const uint32_t k = qt - qh < 32u ? qt - qh : 32u;
    advisory_flush(a, flags, advq, qh, k);
    qh += k;
  }
#endif
  tl_mark(3);
}

// Invariants-only kernel: stage 1 alone, same per-warp TMA ring.
template <bool TMA>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    k_invariants(const double* __restrict__ a, long long n, double* __restrict__ inv,
                 double* /*lam: unused*/, uint8_t* /*flags: unused*/) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpRing R = make_ring(S, a, n, warp, lane);
  const bool inv32 = ((uintptr_t)inv & 31u) == 0;
  if (TMA && lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&R.bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  sched_init(S);
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  ring_prologue<TMA>(R);
  for (uint32_t it = 0;; ++it) {
    int cnt;
    long long c, base;
    double* buf = ring_acquire<TMA>(R, it, c, base, cnt);
    if (!buf) break;
    if (it == 0) ring_kick<TMA>(R);
#pragma unroll
    for (int h = 0; h < kRPL; ++h) {
      if (32 * h >= cnt) {  // half chunk
        if (h == kRPL - 1) ring_release<TMA>(R, c, it, buf);
        continue;
      }
      double m[9];
      bool mod;
      ring_read(buf, lane, h, m, mod);
      if (h == kRPL - 1) ring_release<TMA>(R, c, it, buf);
      const Inv v = invariants_warp(m, mod, 0xffffffffu);
      if (lane + 32 * h < cnt) store_inv(inv, base + 32 * h + lane, v, inv32);
    }
  }
}

static __global__ void __launch_bounds__(kThreads) k_triple_angle(const double* __restrict__ j3,
                                                           const double* __restrict__ disc,
                                                           long long n, double* __restrict__ phi) {
  __shared__ __align__(16) double tab[kTabDoubles + 7];
  load_tables(tab);
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    phi[i] = triple_angle(j3[i], disc[i], tab);
}

}  // namespace eig33b
