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
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/eig33_cuda.h"
#include <cstdlib>

#include "eig33_internal.h"

namespace {

constexpr size_t kChunk = size_t(1) << 22;  // records per chunk (302 MB in, 101 MB out)
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
        (e = cudaMalloc(&s.flags[i], cap)) != cudaSuccess)
      return fail(EIG33_ECUDA, "cudaMalloc staging", e);
  }
  s.cap = cap;
  return EIG33_OK;
}

// Page-locking a caller's pageable buffer per call (cudaHostRegister +
// Unregister) measured slower than the driver's staged pageable copies at every
// size (1 record: 1.1 ms vs 31 us; 2^22 records: 55 vs 48 ms, tools/call_latency.py),
// so by default it is not done; EIG33_PIN_MIN_BYTES=<bytes> re-enables it above
// that size (measurement).  Buffers the caller already pinned are used directly.
size_t pin_min_bytes() {
  static const size_t v = [] {
    const char* e = getenv("EIG33_PIN_MIN_BYTES");
    return e ? (size_t)strtoull(e, nullptr, 10) : ~size_t(0);
  }();
  return v;
}

// Page-lock a host range for the duration of a call unless it already is.
struct PinGuard {
  void* p = nullptr;
  bool registered = false;
  PinGuard(const void* ptr, size_t bytes) {
    if (!ptr || !bytes || bytes < pin_min_bytes()) return;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost) return;
    cudaGetLastError();
    if (cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterPortable) == cudaSuccess) {
      p = const_cast<void*>(ptr);
      registered = true;
    } else {
      cudaGetLastError();  // fall back to pageable copies
    }
  }
  ~PinGuard() {
    if (registered) cudaHostUnregister(p);
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
// of host threads splits a copy into 4 MB parts; the calling thread works too.
// One copy at a time (calls are serialised); never destroyed (threads parked).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool;
    return *p;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < 2 * kPart || nworkers_ == 0) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);
    {
      std::lock_guard<std::mutex> g(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      nparts_ = (bytes + kPart - 1) / kPart;
      finished_.store(0);
      next_.store(0);
      ++gen_;
    }
    cv_.notify_all();
    run_parts();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return finished_.load() == nparts_; });
  }

 private:
  static constexpr size_t kPart = size_t(4) << 20;
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nworkers_ = hw > 1 ? std::min(hw, 16u) - 1 : 0;
    for (unsigned i = 0; i < nworkers_; ++i) std::thread([this] { work(); }).detach();
  }
  void run_parts() {
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= nparts_) return;
      const size_t off = i * kPart, len = std::min(kPart, bytes_ - off);
      std::memcpy(dst_ + off, src_ + off, len);
      if (finished_.fetch_add(1) + 1 == nparts_) {
        std::lock_guard<std::mutex> g(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void work() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
      }
      run_parts();
    }
  }
  unsigned nworkers_ = 0;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, nparts_ = 0;
  std::atomic<size_t> next_{0}, finished_{0};
  unsigned long long gen_ = 0;
};

// Pinned host bounce buffers (per device, grown on demand) for callers whose
// buffers are pageable: the pool copies a chunk into pinned memory while the
// copy engines move the previous chunks, instead of the driver's serial staging.
constexpr size_t kStageChunk = size_t(1) << 20;         // records per staged chunk
constexpr size_t kStageMinBytes = size_t(8) << 20;      // smaller inputs: pageable direct
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
    void *a, *b, *c, *d;
    if ((e = cudaHostAlloc(&a, cap * 9 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&b, cap * 4 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&c, cap * 3 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess ||
        (e = cudaHostAlloc(&d, cap, cudaHostAllocPortable)) != cudaSuccess)
      return fail(EIG33_ECUDA, "cudaHostAlloc staging", e);
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
  auto copy_out = [&](size_t c) -> int {
    const int b = int(c % kSets);
    const size_t lo = c * chunk, cnt = std::min(chunk, n - lo);
    const cudaError_t e = cudaEventSynchronize(h.done[b]);
    if (e != cudaSuccess) return fail(EIG33_ECUDA, "staged D2H", e);
    if (out_inv) pool.copy(h_inv + lo * 4, h.inv[b], cnt * 4 * sizeof(double));
    if (!inv_only(op)) pool.copy(h_lam + lo * 3, h.lam[b], cnt * 3 * sizeof(double));
    if (want_flags) std::memcpy(flags_out + lo, h.fl[b], cnt);
    return EIG33_OK;
  };
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = int(c % kSets);
    cudaStream_t st = s.st[b];
    const size_t lo = c * chunk, cnt = std::min(chunk, n - lo);
    if (c >= (size_t)kSets && (rc = copy_out(c - kSets))) return rc;  // also frees set b
    pool.copy(h.in[b], h_a + lo * 9, cnt * 9 * sizeof(double));
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
    if ((rc = copy_out(c))) return rc;
  return EIG33_OK;
}

int run_device(Op op, const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
               int device, bool* any_notsym) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaSetDevice", e);
  if (n == 0) return EIG33_OK;
  if (device < 0 || device >= 64) return fail(EIG33_EINVAL, "device index out of range");
  Staging& s = g_stage[device];
  std::lock_guard<std::mutex> lock(s.mu);
  const bool want_flags = h_flags != nullptr || op == Op::Sym;
  std::vector<uint8_t> local_flags;
  uint8_t* flags_out = h_flags;
  if (op == Op::Sym && !h_flags) {
    local_flags.resize(n);
    flags_out = local_flags.data();
  }
  int rc;
  // Caller buffers that are pageable and large go through pinned bounce
  // buffers with parallel host copies; pinned ones are DMA'd directly.
  const bool pinned = is_pinned(h_a) && is_pinned(h_inv) && is_pinned(h_lam) && is_pinned(h_flags);
  if (!pinned && n * 9 * sizeof(double) >= kStageMinBytes && pin_min_bytes() == ~size_t(0)) {
    rc = run_staged(op, s, h_a, n, h_inv, h_lam, flags_out, want_flags, device);
    if (rc) return rc;
    if (op == Op::Sym && any_notsym) {
      bool any = false;
      for (size_t i = 0; i < n && !any; ++i) any = (flags_out[i] & EIG33_FLAG_NOT_SYMMETRIC) != 0;
      *any_notsym = any;
    }
    return EIG33_OK;
  }
  const size_t chunk = n < kChunk ? ((n + 1) & ~size_t(1)) : kChunk;
  rc = ensure(s, chunk);
  if (rc) return rc;
  PinGuard pa(h_a, n * 9 * sizeof(double));
  PinGuard pi(h_inv, h_inv ? n * 4 * sizeof(double) : 0);
  PinGuard pl(h_lam, h_lam ? n * 3 * sizeof(double) : 0);
  PinGuard pf(h_flags, h_flags ? n : 0);
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
  if (op == Op::Sym && any_notsym) {
    bool any = false;
    for (size_t i = 0; i < n && !any; ++i) any = (flags_out[i] & EIG33_FLAG_NOT_SYMMETRIC) != 0;
    *any_notsym = any;
  }
  return EIG33_OK;
}

// Contiguous even-aligned shards, one host thread and device each;
// no exchange between devices.  Pageable buffers go through each device's
// staged pipeline (the host copy pool is shared); pinned ones are DMA'd directly.
int run_multi(Op op, const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
              int ngpu, bool* any_notsym) {
  int have = 0;
  cudaError_t e = cudaGetDeviceCount(&have);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaGetDeviceCount", e);
  if (ngpu < 1 || ngpu > have) return fail(EIG33_EINVAL, "ngpu out of range");
  std::vector<int> rcs(ngpu, 0);
  std::vector<char> anys(ngpu, 0);
  std::vector<std::string> errs(ngpu);
  std::vector<std::thread> th;
  for (int g = 0; g < ngpu; ++g) {
    const size_t lo = 2 * ((size_t)g * n / (2 * (size_t)ngpu));
    const size_t hi = g + 1 == ngpu ? n : 2 * ((size_t)(g + 1) * n / (2 * (size_t)ngpu));
    th.emplace_back([=, &rcs, &errs, &anys] {
      bool any = false;
      rcs[g] = run_device(op, h_a + lo * 9, hi - lo, h_inv ? h_inv + lo * 4 : nullptr,
                          h_lam ? h_lam + lo * 3 : nullptr, h_flags ? h_flags + lo : nullptr, g,
                          any_notsym ? &any : nullptr);
      anys[g] = any;
      if (rcs[g]) errs[g] = eig33cu_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int g = 0; g < ngpu; ++g)
    if (rcs[g]) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
  if (any_notsym) {
    *any_notsym = false;
    for (int g = 0; g < ngpu; ++g) *any_notsym = *any_notsym || anys[g];
  }
  return EIG33_OK;
}

}  // namespace

extern "C" {

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
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_eigvalss_host: null pointer");
  bool any = false;
  const int rc = run_device(Op::Sym, h_a, n, h_inv, h_lam, h_flags, device, &any);
  if (rc) return rc;
  return any ? fail(EIG33_ENOTSYM, "matrix is not symmetric to working accuracy") : EIG33_OK;
}

int eig33_multi_eigvals(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                        int ngpu) {
  eig33b::set_error("");
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_multi_eigvals: null pointer");
  return run_multi(Op::Eig, h_a, n, h_inv, h_lam, h_flags, ngpu, nullptr);
}

int eig33_multi_invariants(const double* h_a, size_t n, double* h_inv, int ngpu) {
  eig33b::set_error("");
  if (n && (!h_a || !h_inv)) return fail(EIG33_EINVAL, "eig33_multi_invariants: null pointer");
  return run_multi(Op::Inv, h_a, n, h_inv, nullptr, nullptr, ngpu, nullptr);
}

int eig33_multi_eigvalss(const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
                         int ngpu) {
  eig33b::set_error("");
  if (n && (!h_a || !h_lam)) return fail(EIG33_EINVAL, "eig33_multi_eigvalss: null pointer");
  bool any = false;
  const int rc = run_multi(Op::Sym, h_a, n, h_inv, h_lam, h_flags, ngpu, &any);
  if (rc) return rc;
  return any ? fail(EIG33_ENOTSYM, "matrix is not symmetric to working accuracy") : EIG33_OK;
}

}  // extern "C"
