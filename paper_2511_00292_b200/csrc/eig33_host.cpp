// eig33_host.cpp -- host-buffer entry points of the C ABI (include/eig33_cuda.h):
// chunked H2D -> fused kernel -> D2H pipelines on one device, and the
// multi-GPU shard driver.  No CPU compute path exists here: every record is
// evaluated by the sm_100a kernels in eig33_kernels.cu.
//
// Pipeline: records are cut into chunks of kChunk (even, so every chunk's
// device copy stays 16-B aligned for the TMA loads); chunk c uses buffer set
// c % kSets and stream c % kSets, so H2D of chunk c+1, the kernel of chunk c
// and D2H of chunk c-1 overlap on the two copy engines and the SMs.  Caller
// buffers that are already page-locked are DMA'd directly; large pageable ones
// go through pinned bounce buffers filled and drained by a pool of host threads
// (run_staged); small pageable ones use the driver's staged copies.  Device and
// pinned staging buffers are cached per device and grown on demand.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <initializer_list>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/eig33_cuda.h"
#include <cstdlib>

#include "eig33_internal.h"

namespace {

// Chunk geometry (the CPU pipeline test, tests/test_hostpipe.py, builds with
// small values so that a few thousand records already span many chunks).
#ifndef EIG33_HOST_CHUNK_LOG2
#define EIG33_HOST_CHUNK_LOG2 22
#endif
#ifndef EIG33_STAGE_CHUNK_LOG2
#define EIG33_STAGE_CHUNK_LOG2 20
#endif
#ifndef EIG33_STAGE_MIN_BYTES
#define EIG33_STAGE_MIN_BYTES (size_t(8) << 20)
#endif
constexpr size_t kChunk = size_t(1) << EIG33_HOST_CHUNK_LOG2;  // records per chunk (302 MB in, 101 MB out)
constexpr int kSets = 3;

int fail(int code, const std::string& what, cudaError_t e = cudaSuccess) {
  std::string m = what;
  if (e != cudaSuccess) m += std::string(": ") + cudaGetErrorString(e);
  eig33b::set_error(m);
  return code;
}

struct Staging {
  std::mutex mu;
  size_t cap = 0;
  double* a[kSets] = {};
  double* inv[kSets] = {};
  double* lam[kSets] = {};
  uint8_t* flags[kSets] = {};
  cudaStream_t st[kSets] = {};
  bool streams = false;
};
Staging g_stage[64];

int ensure(Staging& s, size_t cap) {
  cudaError_t e;
  if (!s.streams) {
    for (int i = 0; i < kSets; ++i) {
      e = cudaStreamCreateWithFlags(&s.st[i], cudaStreamNonBlocking);
      if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaStreamCreate", e);
    }
    s.streams = true;
  }
  if (cap <= s.cap) return EIG33_OK;
  for (int i = 0; i < kSets; ++i) {
    cudaFree(s.a[i]);
    cudaFree(s.inv[i]);
    cudaFree(s.lam[i]);
    cudaFree(s.flags[i]);
    s.a[i] = s.inv[i] = s.lam[i] = nullptr;
    s.flags[i] = nullptr;
  }
  s.cap = 0;
  for (int i = 0; i < kSets; ++i) {
    if ((e = cudaMalloc(&s.a[i], cap * 9 * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&s.inv[i], cap * 4 * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&s.lam[i], cap * 3 * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&s.flags[i], cap)) != cudaSuccess) {
      cudaGetLastError();
      return fail(EIG33_ECUDA, "cudaMalloc staging", e);  // cap stays 0: the next call reallocates
    }
  }
  s.cap = cap;
  return EIG33_OK;
}

// Page-locking a caller's pageable buffer per call (cudaHostRegister +
// Unregister) measured slower than the driver's staged pageable copies at every
// size (1 record: 1.1 ms vs 31 us; 2^22 records: 55 vs 48 ms, tools/call_latency.py),
// so it is never done: buffers the caller already pinned are DMA'd directly,
// large pageable ones go through the pinned bounce buffers of run_staged.

// Restores the calling thread's current device on every return path (the
// host entry points switch to the requested device).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Inv* write invariants only (Stable, Naive, NaiveTensor); Eig/Sym write lambda.
enum class Op { Inv, InvNaive, InvTensor, Eig, Sym };
bool inv_only(Op op) { return op == Op::Inv || op == Op::InvNaive || op == Op::InvTensor; }

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost) return true;
  cudaGetLastError();
  return false;
}

// Parallel memcpy for the staged (pageable-buffer) pipeline: a persistent pool
// of host threads splits each copy into 1 MB parts; the calling thread works on
// its own copies too (copy_all: a chunk's outputs and the next input at once).  Several copies may be in flight at once (the multi-GPU
// driver runs one host thread per device): each copy is a Job with its own
// counters, idle workers join any job that still has unclaimed parts, and a
// copy returns only after every part is done AND no worker still holds a
// reference to its Job (so a slow worker can never touch a finished job's
// state or the next job's buffers).  Never destroyed (threads parked).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool;
    return *p;
  }
  struct Span {
    void* dst;
    const void* src;
    size_t bytes;
  };
  void copy(void* dst, const void* src, size_t bytes) { copy_all({Span{dst, src, bytes}}); }
  // Several copies at once (e.g. one chunk's input and an older chunk's
  // outputs): all their parts go to the pool together, the caller works too,
  // and the call returns when every one is complete.
  void copy_all(std::initializer_list<Span> spans) {
    Job jobs[4];
    size_t nj = 0;
    for (const Span& sp : spans) {
      if (sp.bytes == 0) continue;
      if (sp.bytes < 2 * kPart || nworkers_ == 0 || nj == 4) {
        std::memcpy(sp.dst, sp.src, sp.bytes);
        continue;
      }
      Job& j = jobs[nj++];
      j.dst = static_cast<char*>(sp.dst);
      j.src = static_cast<const char*>(sp.src);
      j.bytes = sp.bytes;
      j.nparts = (sp.bytes + kPart - 1) / kPart;
    }
    if (nj == 0) return;
    {
      std::lock_guard<std::mutex> g(mu_);
      for (size_t k = 0; k < nj; ++k) jobs_.push_back(&jobs[k]);
    }
    cv_.notify_all();
    for (size_t k = 0; k < nj; ++k) run(jobs[k]);
    std::unique_lock<std::mutex> g(mu_);
    for (size_t k = 0; k < nj; ++k) {
      Job& j = jobs[k];
      done_cv_.wait(g, [&] { return j.done.load() == j.nparts && j.refs == 0; });
      unlink(&j);
    }
  }

 private:
// 1 MB parts: a 2^20-record chunk's 24-MB lambda copy then spreads over every
// worker (4 MB parts left most of 16 idle: +18% on 2^24 pageable records,
// tools/pageable_rate.py; streaming stores instead of memcpy measured no change)
#ifndef EIG33_COPY_PART
#define EIG33_COPY_PART (size_t(1) << 20)
#endif

  static constexpr size_t kPart = EIG33_COPY_PART;
  struct Job {
    char* dst = nullptr;
    const char* src = nullptr;
    size_t bytes = 0, nparts = 0;
    std::atomic<size_t> next{0}, done{0};
    int refs = 0;  // workers inside run(); guarded by mu_
  };
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nworkers_ = hw > 1 ? std::min(hw, 32u) - 1 : 0;
    for (unsigned i = 0; i < nworkers_; ++i) std::thread([this] { work(); }).detach();
  }
  void run(Job& j) {
    for (;;) {
      const size_t i = j.next.fetch_add(1);
      if (i >= j.nparts) return;
      const size_t off = i * kPart, len = std::min(kPart, j.bytes - off);
      std::memcpy(j.dst + off, j.src + off, len);
      if (j.done.fetch_add(1) + 1 == j.nparts) {
        std::lock_guard<std::mutex> g(mu_);
        done_cv_.notify_all();
      }
    }
  }
  // first listed job with unclaimed parts (mu_ held)
  Job* pick() {
    for (Job* j : jobs_)
      if (j->next.load() < j->nparts) return j;
    return nullptr;
  }
  void unlink(Job* j) {  // mu_ held
    for (size_t k = 0; k < jobs_.size(); ++k)
      if (jobs_[k] == j) {
        jobs_.erase(jobs_.begin() + (long)k);
        return;
      }
  }
  void work() {
    for (;;) {
      Job* j = nullptr;
      {
        // one pick() under the lock: another thread's run() may claim the
        // last parts (an atomic, outside the lock) between two calls
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return (j = pick()) != nullptr; });
        ++j->refs;
      }
      run(*j);
      {
        std::lock_guard<std::mutex> g(mu_);
        --j->refs;
      }
      done_cv_.notify_all();
    }
  }
  unsigned nworkers_ = 0;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<Job*> jobs_;
};

// Pinned host bounce buffers (per device, grown on demand) for callers whose
// buffers are pageable: the pool copies a chunk into pinned memory while the
// copy engines move the previous chunks, instead of the driver's serial staging.
constexpr size_t kStageChunk = size_t(1) << EIG33_STAGE_CHUNK_LOG2;  // records per staged chunk
constexpr size_t kStageMinBytes = EIG33_STAGE_MIN_BYTES;               // smaller inputs: pageable direct
struct HostStaging {
  size_t cap = 0;
  double* in[kSets] = {};
  double* inv[kSets] = {};
  double* lam[kSets] = {};
  uint8_t* fl[kSets] = {};
  cudaEvent_t done[kSets] = {};
};
HostStaging g_hstage[64];

int ensure_host(HostStaging& h, size_t cap) {
  cudaError_t e;
  if (!h.done[0])
    for (int i = 0; i < kSets; ++i)
      if ((e = cudaEventCreateWithFlags(&h.done[i], cudaEventDisableTiming)) != cudaSuccess)
        return fail(EIG33_ECUDA, "cudaEventCreate", e);
  if (cap <= h.cap) return EIG33_OK;
  for (int i = 0; i < kSets; ++i) {
    cudaFreeHost(h.in[i]);
    cudaFreeHost(h.inv[i]);
    cudaFreeHost(h.lam[i]);
    cudaFreeHost(h.fl[i]);
    h.in[i] = h.inv[i] = h.lam[i] = nullptr;
    h.fl[i] = nullptr;
  }
  h.cap = 0;
  for (int i = 0; i < kSets; ++i) {
    void *a = nullptr, *b = nullptr, *c = nullptr, *d = nullptr;
    if ((e = cudaHostAlloc(&a, cap * 9 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&b, cap * 4 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&c, cap * 3 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&d, cap, cudaHostAllocPortable)) != cudaSuccess) {
      for (void* p : {a, b, c, d}) cudaFreeHost(p);  // (the sets before i stay; cap stays 0)
      return fail(EIG33_ECUDA, "cudaHostAlloc staging", e);
    }
    h.in[i] = static_cast<double*>(a);
    h.inv[i] = static_cast<double*>(b);
    h.lam[i] = static_cast<double*>(c);
    h.fl[i] = static_cast<uint8_t*>(d);
  }
  h.cap = cap;
  return EIG33_OK;
}

int launch_op(Op op, const double* d_a, size_t cnt, double* d_inv, double* d_lam, uint8_t* d_fl,
              cudaStream_t st) {
  switch (op) {
    case Op::Inv: return eig33cu_invariants(d_a, cnt, d_inv, st);
    case Op::InvNaive: return eig33cu_invariants_variant(d_a, cnt, 1, d_inv, st);
    case Op::InvTensor: return eig33cu_invariants_variant(d_a, cnt, 2, d_inv, st);
    case Op::Eig: return eig33cu_eigvals(d_a, cnt, d_inv, d_lam, d_fl, st);
    case Op::Sym: return eig33cu_eigvalss(d_a, cnt, d_inv, d_lam, d_fl, st);
  }
  return EIG33_EINVAL;
}

// Waits for everything queued on the device's three pipeline streams; used on
// every error return so that no async copy can still write a caller buffer
// (or read a staging buffer) after the call has returned.
void drain(Staging& s) {
  for (int i = 0; i < kSets; ++i)
    if (s.st[i]) cudaStreamSynchronize(s.st[i]);
  cudaGetLastError();
}

// Index of the first record whose flag byte carries NotSymmetric, or -1.
long long first_notsym(const uint8_t* flags, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (flags[i] & EIG33_FLAG_NOT_SYMMETRIC) return (long long)i;
  return -1;
}

// Staged pipeline: chunk c goes caller -> pinned in[b] (pool copy) -> device
// (H2D) -> kernel -> pinned out[b] (D2H) -> caller (pool copy), b = c % kSets;
// the host copies of chunk c overlap the device work of chunks c-1, c-2.
int run_staged(Op op, Staging& s, const double* h_a, size_t n, double* h_inv, double* h_lam,
               uint8_t* flags_out, bool want_flags, int device) {
  HostStaging& h = g_hstage[device];
  const size_t chunk = std::min(kStageChunk, (n + 1) & ~size_t(1));
  int rc = ensure(s, chunk);
  if (!rc) rc = ensure_host(h, chunk);
  if (rc) return rc;
  CopyPool& pool = CopyPool::get();
  const bool out_inv = h_inv != nullptr;
  const size_t nchunks = (n + chunk - 1) / chunk;
  // copy-out of chunk c (after its D2H), together with the copy-in of the
  // chunk that reuses its set (nxt < n), in one pool round
  auto copy_out = [&](size_t c, size_t nxt) -> int {
    const int b = int(c % kSets);
    const size_t lo = c * chunk, cnt = std::min(chunk, n - lo);
    const cudaError_t e = cudaEventSynchronize(h.done[b]);
    if (e != cudaSuccess) return fail(EIG33_ECUDA, "staged D2H", e);
    const size_t ilo = nxt * chunk, icnt = nxt < nchunks ? std::min(chunk, n - ilo) : 0;
    pool.copy_all({{out_inv ? h_inv + lo * 4 : nullptr, h.inv[b], out_inv ? cnt * 4 * sizeof(double) : 0},
                   {inv_only(op) ? nullptr : h_lam + lo * 3, h.lam[b], inv_only(op) ? 0 : cnt * 3 * sizeof(double)},
                   {h.in[b], icnt ? h_a + ilo * 9 : h_a, icnt * 9 * sizeof(double)}});
    if (want_flags) std::memcpy(flags_out + lo, h.fl[b], cnt);
    return EIG33_OK;
  };
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = int(c % kSets);
    cudaStream_t st = s.st[b];
    const size_t lo = c * chunk, cnt = std::min(chunk, n - lo);
    if (c >= (size_t)kSets) {  // frees set b and fills its input with chunk c
      if ((rc = copy_out(c - kSets, c))) return rc;
    } else {
      pool.copy(h.in[b], h_a + lo * 9, cnt * 9 * sizeof(double));
    }
    cudaError_t e = cudaMemcpyAsync(s.a[b], h.in[b], cnt * 9 * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(EIG33_ECUDA, "H2D", e);
    rc = launch_op(op, s.a[b], cnt, out_inv ? s.inv[b] : nullptr, s.lam[b],
                   want_flags ? s.flags[b] : nullptr, st);
    if (rc) return fail(rc, eig33cu_last_error());
    if (out_inv && (e = cudaMemcpyAsync(h.inv[b], s.inv[b], cnt * 4 * sizeof(double),
                                        cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return fail(EIG33_ECUDA, "D2H inv", e);
    if (!inv_only(op) && (e = cudaMemcpyAsync(h.lam[b], s.lam[b], cnt * 3 * sizeof(double),
                                              cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return fail(EIG33_ECUDA, "D2H lam", e);
    if (want_flags && (e = cudaMemcpyAsync(h.fl[b], s.flags[b], cnt, cudaMemcpyDeviceToHost, st)) !=
                          cudaSuccess)
      return fail(EIG33_ECUDA, "D2H flags", e);
    if ((e = cudaEventRecord(h.done[b], st)) != cudaSuccess) return fail(EIG33_ECUDA, "event", e);
  }
  for (size_t c = nchunks > (size_t)kSets ? nchunks - kSets : 0; c < nchunks; ++c)
    if ((rc = copy_out(c, nchunks))) return rc;
  return EIG33_OK;
}

// Direct pipeline over caller buffers (pinned, or small pageable ones the
// driver stages itself): H2D of chunk c+1, kernel of chunk c and D2H of chunk
// c-1 overlap on the three streams.
int run_direct(Op op, Staging& s, const double* h_a, size_t n, double* h_inv, double* h_lam,
               uint8_t* flags_out, bool want_flags) {
  const size_t chunk = n < kChunk ? ((n + 1) & ~size_t(1)) : kChunk;
  int rc = ensure(s, chunk);
  if (rc) return rc;
  cudaError_t e;
  const size_t nchunks = (n + chunk - 1) / chunk;
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = int(c % kSets);
    cudaStream_t st = s.st[b];
    const size_t lo = c * chunk, cnt = (n - lo) < chunk ? (n - lo) : chunk;
    e = cudaMemcpyAsync(s.a[b], h_a + lo * 9, cnt * 9 * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(EIG33_ECUDA, "H2D", e);
    double* dinv = h_inv ? s.inv[b] : nullptr;
    uint8_t* dfl = want_flags ? s.flags[b] : nullptr;
    rc = launch_op(op, s.a[b], cnt, inv_only(op) ? s.inv[b] : dinv, s.lam[b], dfl, st);
    if (rc) return fail(rc, eig33cu_last_error());
    if (h_inv || inv_only(op)) {
      e = cudaMemcpyAsync(h_inv + lo * 4, s.inv[b], cnt * 4 * sizeof(double), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return fail(EIG33_ECUDA, "D2H inv", e);
    }
    if (!inv_only(op)) {
      e = cudaMemcpyAsync(h_lam + lo * 3, s.lam[b], cnt * 3 * sizeof(double), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return fail(EIG33_ECUDA, "D2H lam", e);
      if (want_flags) {
        e = cudaMemcpyAsync(flags_out + lo, s.flags[b], cnt, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fail(EIG33_ECUDA, "D2H flags", e);
      }
    }
  }
  for (int i = 0; i < kSets; ++i) {
    e = cudaStreamSynchronize(s.st[i]);
    if (e != cudaSuccess) return fail(EIG33_ECUDA, "stream sync", e);
  }
  return EIG33_OK;
}

// One device, synchronous.  *notsym (eigvalss) receives the first record that
// failed the symmetry gate, or -1.  The caller's current device is restored.
int run_device(Op op, const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
               int device, long long* notsym) {
  if (notsym) *notsym = -1;
  if (n == 0) return EIG33_OK;
  int have = 0;
  if (cudaGetDeviceCount(&have) != cudaSuccess) have = 0;
  if (device < 0 || device >= 64 || device >= have) return fail(EIG33_EINVAL, "device index out of range");
  DeviceGuard keep;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaSetDevice", e);
  Staging& s = g_stage[device];
  std::lock_guard<std::mutex> lock(s.mu);
  const bool want_flags = h_flags != nullptr || op == Op::Sym;
  std::vector<uint8_t> local_flags;
  uint8_t* flags_out = h_flags;
  if (op == Op::Sym && !h_flags) {
    local_flags.resize(n);
    flags_out = local_flags.data();
  }
  // Caller buffers that are pageable and large go through pinned bounce
  // buffers with parallel host copies; pinned ones are DMA'd directly.
  const bool pinned = is_pinned(h_a) && is_pinned(h_inv) && is_pinned(h_lam) && is_pinned(h_flags);
  const int rc = (!pinned && n * 9 * sizeof(double) >= kStageMinBytes)
                     ? run_staged(op, s, h_a, n, h_inv, h_lam, flags_out, want_flags, device)
                     : run_direct(op, s, h_a, n, h_inv, h_lam, flags_out, want_flags);
  if (rc) {
    drain(s);
    return rc;
  }
  if (op == Op::Sym && notsym) *notsym = first_notsym(flags_out, n);
  return EIG33_OK;
}

// Contiguous even-aligned shards, one host thread and device each;
// no exchange between devices.  Pageable buffers go through each device's
// staged pipeline (the host copy pool serves all devices at once); pinned ones
// are DMA'd directly.  `devices` lists the device of each shard (a device may
// repeat: its shards then take turns on its pipeline).
int run_multi(Op op, const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
              const int* devices, int ndev, long long* notsym) {
  if (notsym) *notsym = -1;
  int have = 0;
  cudaError_t e = cudaGetDeviceCount(&have);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaGetDeviceCount", e);
  if (ndev < 1 || ndev > 64) return fail(EIG33_EINVAL, "ngpu out of range");
  for (int g = 0; g < ndev; ++g)
    if (devices[g] < 0 || devices[g] >= have) return fail(EIG33_EINVAL, "device index out of range");
  std::vector<int> rcs(ndev, 0);
  std::vector<long long> bad(ndev, -1);
  std::vector<std::string> errs(ndev);
  std::vector<std::thread> th;
  std::vector<size_t> los(ndev);
  for (int g = 0; g < ndev; ++g) {
    const size_t lo = 2 * ((size_t)g * n / (2 * (size_t)ndev));
    const size_t hi = g + 1 == ndev ? n : 2 * ((size_t)(g + 1) * n / (2 * (size_t)ndev));
    los[g] = lo;
    const int dev = devices[g];
    th.emplace_back([=, &rcs, &errs, &bad] {
      rcs[g] = run_device(op, h_a + lo * 9, hi - lo, h_inv ? h_inv + lo * 4 : nullptr,
                          h_lam ? h_lam + lo * 3 : nullptr, h_flags ? h_flags + lo : nullptr, dev,
                          notsym ? &bad[g] : nullptr);
      if (rcs[g]) errs[g] = eig33cu_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int g = 0; g < ndev; ++g)
    if (rcs[g]) return fail(rcs[g], "shard " + std::to_string(g) + " (device " + std::to_string(devices[g]) +
                                        "): " + errs[g]);
  if (notsym)
    for (int g = 0; g < ndev; ++g)
      if (bad[g] >= 0) {
        *notsym = (long long)los[g] + bad[g];
        break;
      }
  return EIG33_OK;
}

int run_multi_n(Op op, const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                int ngpu, long long* notsym) {
  if (ngpu < 1 || ngpu > 64) return fail(EIG33_EINVAL, "ngpu out of range");
  int have = 0;
  cudaError_t e = cudaGetDeviceCount(&have);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaGetDeviceCount", e);
  if (ngpu > have) return fail(EIG33_EINVAL, "ngpu out of range");
  std::vector<int> devs(ngpu);
  for (int g = 0; g < ngpu; ++g) devs[g] = g;
  return run_multi(op, h_a, n, h_inv, h_lam, h_flags, devs.data(), ngpu, notsym);
}

thread_local long long g_notsym = -1;

int notsym_status(long long first) {
  g_notsym = first;
  if (first < 0) return EIG33_OK;
  return fail(EIG33_ENOTSYM, "matrix is not symmetric to working accuracy (first at record " +
                                 std::to_string(first) + ")");
}

}  // namespace

extern "C" {

long long eig33cu_last_notsym_index(void) { return g_notsym; }

int eig33_invariants_host(const double* h_a, size_t n, double* h_inv, int device) {
  eig33b::set_error("");
  if (n && (!h_a || !h_inv)) return fail(EIG33_EINVAL, "eig33_invariants_host: null pointer");
  return run_device(Op::Inv, h_a, n, h_inv, nullptr, nullptr, device, nullptr);
}

int eig33_invariants_variant_host(const double* h_a, size_t n, int variant, double* h_inv,
                                  int device) {
  eig33b::set_error("");
  if (n && (!h_a || !h_inv)) return fail(EIG33_EINVAL, "eig33_invariants_variant_host: null pointer");
  if (variant < 0 || variant > 2) return fail(EIG33_EINVAL, "eig33_invariants_variant_host: bad variant");
  const Op op = variant == 0 ? Op::Inv : variant == 1 ? Op::InvNaive : Op::InvTensor;
  return run_device(op, h_a, n, h_inv, nullptr, nullptr, device, nullptr);
}

int eig33_eigvals_host(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                       int device) {
  eig33b::set_error("");
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_eigvals_host: null pointer");
  return run_device(Op::Eig, h_a, n, h_inv, h_lam, h_flags, device, nullptr);
}

int eig33_eigvalss_host(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                        int device) {
  eig33b::set_error("");
  g_notsym = -1;
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_eigvalss_host: null pointer");
  long long first = -1;
  const int rc = run_device(Op::Sym, h_a, n, h_inv, h_lam, h_flags, device, &first);
  if (rc) return rc;
  return notsym_status(first);
}

int eig33_multi_eigvals(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                        int ngpu) {
  eig33b::set_error("");
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_multi_eigvals: null pointer");
  return run_multi_n(Op::Eig, h_a, n, h_inv, h_lam, h_flags, ngpu, nullptr);
}

int eig33_multi_eigvals_on(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                           const int* devices, int ndev) {
  eig33b::set_error("");
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_multi_eigvals_on: null pointer");
  if (!devices) return fail(EIG33_EINVAL, "eig33_multi_eigvals_on: null device list");
  return run_multi(Op::Eig, h_a, n, h_inv, h_lam, h_flags, devices, ndev, nullptr);
}

int eig33_multi_invariants(const double* h_a, size_t n, double* h_inv, int ngpu) {
  eig33b::set_error("");
  if (n && (!h_a || !h_inv)) return fail(EIG33_EINVAL, "eig33_multi_invariants: null pointer");
  return run_multi_n(Op::Inv, h_a, n, h_inv, nullptr, nullptr, ngpu, nullptr);
}

int eig33_multi_eigvalss(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                         int ngpu) {
  eig33b::set_error("");
  g_notsym = -1;
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_multi_eigvalss: null pointer");
  long long first = -1;
  const int rc = run_multi_n(Op::Sym, h_a, n, h_inv, h_lam, h_flags, ngpu, &first);
  if (rc) return rc;
  return notsym_status(first);
}

}  // extern "C"
