// eig33_host.cpp -- host-buffer entry points of the C ABI (include/eig33_cuda.h):
// chunked H2D -> fused kernel -> D2H pipelines on one device, and the
// multi-GPU shard driver.  No CPU compute path exists here: every record is
// evaluated by the sm_100a kernels in eig33_kernels.cu.
//
// Pipeline: records are cut into chunks of kChunk (even, so every chunk's
// device copy stays 16-B aligned for the TMA loads); chunk c uses buffer set
// c % kSets and stream c % kSets, so H2D of chunk c+1, the kernel of chunk c
// and D2H of chunk c-1 overlap on the two copy engines and the SMs.  Host
// buffers that are not already page-locked are registered for the duration of
// the call.  Device buffers are cached per device and grown on demand.
#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/eig33_cuda.h"
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

// Page-lock a host range for the duration of a call unless it already is.
struct PinGuard {
  void* p = nullptr;
  bool registered = false;
  PinGuard(const void* ptr, size_t bytes) {
    if (!ptr || !bytes) return;
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

enum class Op { Inv, Eig, Sym };

int run_device(Op op, const double* h_a, size_t n, double* h_inv, double* h_lam, uint8_t* h_flags,
               int device, bool* any_notsym) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaSetDevice", e);
  if (n == 0) return EIG33_OK;
  if (device < 0 || device >= 64) return fail(EIG33_EINVAL, "device index out of range");
  Staging& s = g_stage[device];
  std::lock_guard<std::mutex> lock(s.mu);
  const size_t chunk = n < kChunk ? ((n + 1) & ~size_t(1)) : kChunk;
  int rc = ensure(s, chunk);
  if (rc) return rc;
  PinGuard pa(h_a, n * 9 * sizeof(double));
  PinGuard pi(h_inv, h_inv ? n * 4 * sizeof(double) : 0);
  PinGuard pl(h_lam, h_lam ? n * 3 * sizeof(double) : 0);
  PinGuard pf(h_flags, h_flags ? n : 0);
  const bool want_flags = h_flags != nullptr || op == Op::Sym;
  std::vector<uint8_t> local_flags;
  uint8_t* flags_out = h_flags;
  if (op == Op::Sym && !h_flags) {
    local_flags.resize(n);
    flags_out = local_flags.data();
  }
  const size_t nchunks = (n + chunk - 1) / chunk;
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = int(c % kSets);
    cudaStream_t st = s.st[b];
    const size_t lo = c * chunk, cnt = (n - lo) < chunk ? (n - lo) : chunk;
    e = cudaMemcpyAsync(s.a[b], h_a + lo * 9, cnt * 9 * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(EIG33_ECUDA, "H2D", e);
    double* dinv = h_inv ? s.inv[b] : nullptr;
    uint8_t* dfl = want_flags ? s.flags[b] : nullptr;
    switch (op) {
      case Op::Inv: rc = eig33cu_invariants(s.a[b], cnt, s.inv[b], st); break;
      case Op::Eig: rc = eig33cu_eigvals(s.a[b], cnt, dinv, s.lam[b], dfl, st); break;
      case Op::Sym: rc = eig33cu_eigvalss(s.a[b], cnt, dinv, s.lam[b], dfl, st); break;
    }
    if (rc) return fail(rc, eig33cu_last_error());
    if (h_inv || op == Op::Inv) {
      e = cudaMemcpyAsync(h_inv + lo * 4, s.inv[b], cnt * 4 * sizeof(double), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return fail(EIG33_ECUDA, "D2H inv", e);
    }
    if (op != Op::Inv) {
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

}  // namespace

extern "C" {

int eig33_invariants_host(const double* h_a, size_t n, double* h_inv, int device) {
  eig33b::set_error("");
  if (n && (!h_a || !h_inv)) return fail(EIG33_EINVAL, "eig33_invariants_host: null pointer");
  return run_device(Op::Inv, h_a, n, h_inv, nullptr, nullptr, device, nullptr);
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
  int have = 0;
  cudaError_t e = cudaGetDeviceCount(&have);
  if (e != cudaSuccess) return fail(EIG33_ECUDA, "cudaGetDeviceCount", e);
  if (ngpu < 1 || ngpu > have) return fail(EIG33_EINVAL, "ngpu out of range");
  // Page-lock the whole buffers once (portable: every device sees them pinned).
  // Left to the per-device calls, shard boundaries that share a page would make
  // all but the first registration fail and fall back to pageable copies.
  const PinGuard pin_a(h_a, n * 9 * sizeof(double));
  const PinGuard pin_l(h_lam, n * 3 * sizeof(double));
  const PinGuard pin_i(h_inv, h_inv ? n * 4 * sizeof(double) : 0);
  const PinGuard pin_f(h_flags, h_flags ? n : 0);
  std::vector<int> rcs(ngpu, 0);
  std::vector<std::string> errs(ngpu);
  std::vector<std::thread> th;
  for (int g = 0; g < ngpu; ++g) {
    const size_t lo = 2 * ((size_t)g * n / (2 * (size_t)ngpu));
    const size_t hi = g + 1 == ngpu ? n : 2 * ((size_t)(g + 1) * n / (2 * (size_t)ngpu));
    th.emplace_back([=, &rcs, &errs] {
      rcs[g] = run_device(Op::Eig, h_a + lo * 9, hi - lo, h_inv ? h_inv + lo * 4 : nullptr,
                          h_lam + lo * 3, h_flags ? h_flags + lo : nullptr, g, nullptr);
      if (rcs[g]) errs[g] = eig33cu_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int g = 0; g < ngpu; ++g)
    if (rcs[g]) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
  return EIG33_OK;
}

}  // extern "C"
