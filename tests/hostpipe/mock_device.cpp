// mock_device.cpp -- TEST INFRASTRUCTURE: the mock CUDA runtime of
// mock/cuda_runtime.h plus CPU stand-ins for the device-pointer entry points
// eig33_host.cpp launches (eig33cu_invariants / _variant, eig33cu_eigvals,
// eig33cu_eigvalss), computed with the product's own per-record math built
// for the CPU (eig33_math.cuh), so the host pipeline's outputs can be checked
// bit for bit without a GPU.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <set>
#include <string>

#include "mock/cuda_runtime.h"
#define EIG33_TABLE_DECL static const
#include "../../paper_2511_00292_b200/csrc/eig33_tables.h"
#include "../../paper_2511_00292_b200/csrc/eig33_math.cuh"
#include "../../include/eig33_cuda.h"
#include "../../paper_2511_00292_b200/csrc/eig33_internal.h"

namespace {
struct Alloc {
  size_t bytes;
  int device;  // -1: pinned host
};
std::mutex g_mu;
std::map<const char*, Alloc> g_allocs;
thread_local int g_cur = 0;
thread_local std::string g_err;
int g_launches = 0;

int env_int(const char* k, int dflt) {
  const char* v = getenv(k);
  return v ? atoi(v) : dflt;
}
[[noreturn]] void die(const char* what) {
  fprintf(stderr, "MOCK FAULT: %s\n", what);
  abort();
}
// allocation containing [p, p+bytes), or nullptr
const Alloc* find(const void* p, size_t bytes, const char** base = nullptr) {
  std::lock_guard<std::mutex> g(g_mu);
  const char* c = static_cast<const char*>(p);
  auto it = g_allocs.upper_bound(c);
  if (it == g_allocs.begin()) return nullptr;
  --it;
  if (c < it->first || c + bytes > it->first + it->second.bytes) return nullptr;
  if (base) *base = it->first;
  return &it->second;
}
void check_dev(const void* p, size_t bytes, const char* what) {
  if (!p || !bytes) return;
  const Alloc* a = find(p, bytes);
  if (!a || a->device < 0) die(what);
  if (a->device != g_cur) die("kernel buffer on another device than the current one");
}
}  // namespace

struct MockStream {
  int device;
};
struct MockEvent {
  int device;
};

const char* cudaGetErrorString(cudaError_t e) { return e == cudaSuccess ? "no error" : "mock error"; }
cudaError_t cudaGetLastError(void) { return cudaSuccess; }
cudaError_t cudaGetDevice(int* d) {
  *d = g_cur;
  return cudaSuccess;
}
cudaError_t cudaSetDevice(int d) {
  if (d < 0 || d >= env_int("MOCK_NDEV", 2)) return cudaErrorInvalidDevice;
  g_cur = d;
  return cudaSuccess;
}
cudaError_t cudaGetDeviceCount(int* n) {
  *n = env_int("MOCK_NDEV", 2);
  return cudaSuccess;
}
cudaError_t cudaMalloc(void** p, size_t bytes) {
  char* m = static_cast<char*>(malloc(bytes ? bytes : 1));
  memset(m, 0xA5, bytes);  // garbage, like fresh device memory
  std::lock_guard<std::mutex> g(g_mu);
  g_allocs[m] = Alloc{bytes, g_cur};
  *p = m;
  return cudaSuccess;
}
cudaError_t cudaFree(void* p) {
  if (!p) return cudaSuccess;
  std::lock_guard<std::mutex> g(g_mu);
  if (!g_allocs.erase(static_cast<char*>(p))) die("cudaFree of an unknown pointer");
  free(p);
  return cudaSuccess;
}
cudaError_t cudaHostAlloc(void** p, size_t bytes, unsigned) {
  char* m = static_cast<char*>(malloc(bytes ? bytes : 1));
  std::lock_guard<std::mutex> g(g_mu);
  g_allocs[m] = Alloc{bytes, -1};
  *p = m;
  return cudaSuccess;
}
cudaError_t cudaFreeHost(void* p) { return cudaFree(p); }
cudaError_t cudaStreamCreateWithFlags(cudaStream_t* s, unsigned) {
  *s = new MockStream{g_cur};
  return cudaSuccess;
}
cudaError_t cudaStreamSynchronize(cudaStream_t) { return cudaSuccess; }
cudaError_t cudaEventCreateWithFlags(cudaEvent_t* e, unsigned) {
  *e = new MockEvent{g_cur};
  return cudaSuccess;
}
cudaError_t cudaEventRecord(cudaEvent_t e, cudaStream_t s) {
  if (!e || !s) die("event record on a null handle");
  return cudaSuccess;
}
cudaError_t cudaEventSynchronize(cudaEvent_t e) {
  if (!e) die("event sync on a null handle");
  return cudaSuccess;
}
cudaError_t cudaMemcpyAsync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
  if (!s) die("copy on a null stream");
  if (s->device != g_cur) die("copy on a stream of another device");
  const void* dev = kind == cudaMemcpyHostToDevice ? dst : src;
  check_dev(dev, bytes, kind == cudaMemcpyHostToDevice ? "H2D destination out of bounds"
                                                      : "D2H source out of bounds");
  const void* host = kind == cudaMemcpyHostToDevice ? src : dst;
  const Alloc* h = find(host, 1);
  if (h && h->device >= 0) die("host side of a copy is device memory");
  if (h && !find(host, bytes)) die("pinned host side of a copy out of bounds");
  memcpy(dst, src, bytes);
  return cudaSuccess;
}
cudaError_t cudaPointerGetAttributes(cudaPointerAttributes* a, const void* p) {
  const Alloc* al = find(p, 1);
  a->type = !al ? cudaMemoryTypeUnregistered : al->device < 0 ? cudaMemoryTypeHost : cudaMemoryTypeDevice;
  a->device = al ? al->device : -1;
  return cudaSuccess;
}

// ---- the product's error slot and the device-pointer entry points ----
namespace eig33b {
void set_error(const std::string& m) { g_err = m; }
}  // namespace eig33b

using namespace eig33b;

static int launch_guard() {
  std::lock_guard<std::mutex> g(g_mu);
  ++g_launches;
  const int fail_at = env_int("MOCK_FAIL_LAUNCH_AT", 0);
  if (fail_at && g_launches == fail_at) {  // once per mock_reset()
    g_err = "mock launch failure";
    return EIG33_ECUDA;
  }
  return EIG33_OK;
}

extern "C" {
const char* eig33cu_last_error(void) { return g_err.c_str(); }
int mock_launches(void) { return g_launches; }
void mock_reset(void) { g_launches = 0; }
int mock_live_device_bytes(void) {
  std::lock_guard<std::mutex> g(g_mu);
  size_t b = 0;
  for (auto& kv : g_allocs) b += kv.second.bytes;
  return (int)(b >> 20);
}

int eig33cu_invariants_variant(const double* d_a, size_t n, int variant, double* d_inv, void*) {
  check_dev(d_a, n * 72, "kernel input out of bounds");
  check_dev(d_inv, n * 32, "kernel inv out of bounds");
  if (int rc = launch_guard()) return rc;
  for (size_t i = 0; i < n; ++i) {
    const Inv v = invariants_variant(d_a + 9 * i, variant);
    d_inv[4 * i] = v.i1; d_inv[4 * i + 1] = v.j2; d_inv[4 * i + 2] = v.j3; d_inv[4 * i + 3] = v.disc;
  }
  return EIG33_OK;
}
int eig33cu_invariants(const double* d_a, size_t n, double* d_inv, void* st) {
  return eig33cu_invariants_variant(d_a, n, 0, d_inv, st);
}
static int eig_common(const double* d_a, size_t n, double* d_inv, double* d_lam, uint8_t* d_flags, bool sym) {
  check_dev(d_a, n * 72, "kernel input out of bounds");
  check_dev(d_inv, n * 32, "kernel inv out of bounds");
  check_dev(d_lam, n * 24, "kernel lam out of bounds");
  check_dev(d_flags, n, "kernel flags out of bounds");
  if (int rc = launch_guard()) return rc;
  for (size_t i = 0; i < n; ++i) {
    double m[9];
    memcpy(m, d_a + 9 * i, sizeof m);
    uint8_t f = 0;
    Inv v;
    Lam l;
    if (sym && not_symmetric(m)) {
      f = EIG33_FLAG_NOT_SYMMETRIC;
      const double q = __builtin_nan("");
      v = Inv{q, q, q, q};
      l = Lam{q, q, q};
    } else {
      if (sym) {
        m[3] = m[1];
        m[6] = m[2];
        m[7] = m[5];
      }
      v = invariants(m);
      l = from_invariants(m, v, eig33_tab);
      if (!sym && advisory(m, v)) f = EIG33_FLAG_ADVISORY;
    }
    if (d_inv) {
      d_inv[4 * i] = v.i1; d_inv[4 * i + 1] = v.j2; d_inv[4 * i + 2] = v.j3; d_inv[4 * i + 3] = v.disc;
    }
    d_lam[3 * i] = l.l1; d_lam[3 * i + 1] = l.l2; d_lam[3 * i + 2] = l.l3;
    if (d_flags) d_flags[i] = f;
  }
  return EIG33_OK;
}
int eig33cu_eigvals(const double* d_a, size_t n, double* d_inv, double* d_lam, uint8_t* d_flags, void*) {
  return eig_common(d_a, n, d_inv, d_lam, d_flags, false);
}
int eig33cu_eigvalss(const double* d_a, size_t n, double* d_inv, double* d_lam, uint8_t* d_flags, void*) {
  return eig_common(d_a, n, d_inv, d_lam, d_flags, true);
}
// single-record reference for the checks (same math, no pipeline)
void mock_expected(const double* a, size_t n, double* inv, double* lam, uint8_t* flags, int sym) {
  for (size_t i = 0; i < n; ++i) {
    double m[9];
    memcpy(m, a + 9 * i, sizeof m);
    uint8_t f = 0;
    Inv v;
    Lam l;
    if (sym && not_symmetric(m)) {
      const double q = __builtin_nan("");
      v = Inv{q, q, q, q};
      l = Lam{q, q, q};
      f = EIG33_FLAG_NOT_SYMMETRIC;
    } else {
      if (sym) { m[3] = m[1]; m[6] = m[2]; m[7] = m[5]; }
      v = invariants(m);
      l = from_invariants(m, v, eig33_tab);
      if (!sym && advisory(m, v)) f = EIG33_FLAG_ADVISORY;
    }
    inv[4 * i] = v.i1; inv[4 * i + 1] = v.j2; inv[4 * i + 2] = v.j3; inv[4 * i + 3] = v.disc;
    lam[3 * i] = l.l1; lam[3 * i + 1] = l.l2; lam[3 * i + 2] = l.l3;
    flags[i] = f;
  }
}
// mock pinned allocation for the tests' "pinned caller buffer" cases
void* mock_host_alloc(size_t bytes) {
  void* p = nullptr;
  cudaHostAlloc(&p, bytes, 0);
  return p;
}
void mock_host_free(void* p) { cudaFreeHost(p); }
}  // extern "C"
