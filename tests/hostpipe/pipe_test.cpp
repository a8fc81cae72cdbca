// pipe_test.cpp -- TEST INFRASTRUCTURE: drives the product's host pipeline
// (eig33_host.cpp, compiled against the mock runtime) through every host
// entry point and checks each output bit for bit against the same per-record
// math evaluated directly.  Built with AddressSanitizer by tests/test_hostpipe.py.
//   pipe_test basic | multi | fail | device
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/eig33_cuda.h"
#include "mock/cuda_runtime.h"

extern "C" {
void mock_expected(const double* a, size_t n, double* inv, double* lam, uint8_t* flags, int sym);
void* mock_host_alloc(size_t bytes);
void mock_host_free(void* p);
int mock_launches(void);
void mock_reset(void);
}

static int g_fail = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    if (!(c)) {                                                           \
      fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)

static bool same(const double* x, const double* y, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t a, b;
    memcpy(&a, x + i, 8);
    memcpy(&b, y + i, 8);
    if (a != b && !(std::isnan(x[i]) && std::isnan(y[i]))) return false;
  }
  return true;
}

struct Batch {
  size_t n;
  bool pinned;
  double *a, *inv, *lam;
  uint8_t* fl;
  std::vector<double> va, vinv, vlam;
  std::vector<uint8_t> vfl;
  Batch(size_t n_, bool pinned_, bool sym, uint64_t seed) : n(n_), pinned(pinned_) {
    if (pinned) {
      a = static_cast<double*>(mock_host_alloc(n * 72 + 8));
      inv = static_cast<double*>(mock_host_alloc(n * 32 + 8));
      lam = static_cast<double*>(mock_host_alloc(n * 24 + 8));
      fl = static_cast<uint8_t*>(mock_host_alloc(n + 8));
    } else {
      va.resize(n * 9 + 1);
      vinv.resize(n * 4 + 1);
      vlam.resize(n * 3 + 1);
      vfl.resize(n + 1);
      a = va.data();
      inv = vinv.data();
      lam = vlam.data();
      fl = vfl.data();
    }
    uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
    for (size_t i = 0; i < n * 9; ++i) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      a[i] = ((double)(s >> 11) * 0x1p-53 - 0.5) * ((i % 7) ? 2.0 : 1e-3);
    }
    if (sym)
      for (size_t i = 0; i < n; ++i) {
        a[9 * i + 3] = a[9 * i + 1];
        a[9 * i + 6] = a[9 * i + 2];
        a[9 * i + 7] = a[9 * i + 5];
      }
  }
  ~Batch() {
    if (pinned) {
      mock_host_free(a);
      mock_host_free(inv);
      mock_host_free(lam);
      mock_host_free(fl);
    }
  }
};

static void expect(const Batch& b, int sym, bool want_inv, bool want_fl) {
  std::vector<double> inv(b.n * 4), lam(b.n * 3);
  std::vector<uint8_t> fl(b.n);
  mock_expected(b.a, b.n, inv.data(), lam.data(), fl.data(), sym);
  CHECK(same(b.lam, lam.data(), b.n * 3));
  if (want_inv) CHECK(same(b.inv, inv.data(), b.n * 4));
  if (want_fl) CHECK(memcmp(b.fl, fl.data(), b.n) == 0);
}

static void basic() {
  // built with 2^10-record direct chunks, 2^8-record staged chunks and staging
  // from 64 KB on: these sizes cover one / several / ragged chunks of both paths
  const size_t sizes[] = {1, 2, 3, 255, 1001, 3 * 1024 + 5, 9000};
  for (size_t n : sizes)
    for (int pinned = 0; pinned < 2; ++pinned) {
      Batch b(n, pinned, false, n + pinned);
      CHECK(eig33_eigvals_host(b.a, n, b.inv, b.lam, b.fl, 0) == EIG33_OK);
      expect(b, 0, true, true);
      CHECK(eig33_eigvals_host(b.a, n, nullptr, b.lam, nullptr, 1) == EIG33_OK);
      expect(b, 0, false, false);
      std::vector<double> inv(n * 4);
      CHECK(eig33_invariants_host(b.a, n, b.inv, 0) == EIG33_OK);
      expect(b, 0, true, false);
      CHECK(eig33_invariants_variant_host(b.a, n, 2, inv.data(), 1) == EIG33_OK);
      // eigvalss: symmetric batch ok, then one asymmetric record -> ENOTSYM + its index
      Batch s(n, pinned, true, n * 3 + pinned);
      CHECK(eig33_eigvalss_host(s.a, n, s.inv, s.lam, s.fl, 0) == EIG33_OK);
      CHECK(eig33cu_last_notsym_index() == -1);
      expect(s, 1, true, true);
      const size_t bad = n / 2;
      s.a[9 * bad + 1] += 0.5;
      if (n > 4) s.a[9 * (n - 1) + 2] += 0.5;
      CHECK(eig33_eigvalss_host(s.a, n, nullptr, s.lam, nullptr, 1) == EIG33_ENOTSYM);
      CHECK(eig33cu_last_notsym_index() == (long long)bad);
      CHECK(strstr(eig33cu_last_error(), ("record " + std::to_string(bad)).c_str()) != nullptr);
      expect(s, 1, false, false);
    }
}

static void multi() {
  const size_t n = 2 * 4096 + 77;
  for (int pinned = 0; pinned < 2; ++pinned) {
    Batch b(n, pinned, false, 5 + pinned);
    CHECK(eig33_multi_eigvals(b.a, n, b.inv, b.lam, b.fl, 2) == EIG33_OK);
    expect(b, 0, true, true);
    const int devs[] = {0, 1, 1, 0, 0};
    memset(b.lam, 0, n * 24);
    CHECK(eig33_multi_eigvals_on(b.a, n, b.inv, b.lam, b.fl, devs, 5) == EIG33_OK);
    expect(b, 0, true, true);
    CHECK(eig33_multi_invariants(b.a, n, b.inv, 2) == EIG33_OK);
    expect(b, 0, true, false);
    CHECK(eig33_multi_eigvals(b.a, n, b.inv, b.lam, b.fl, 3) == EIG33_EINVAL);
    const int bad_dev[] = {0, 2};
    CHECK(eig33_multi_eigvals_on(b.a, n, b.inv, b.lam, b.fl, bad_dev, 2) == EIG33_EINVAL);
    Batch s(n, pinned, true, 9 + pinned);
    CHECK(eig33_multi_eigvalss(s.a, n, nullptr, s.lam, nullptr, 2) == EIG33_OK);
    expect(s, 1, false, false);
    s.a[9 * (n - 3) + 5] += 1.0;  // in the last shard
    CHECK(eig33_multi_eigvalss(s.a, n, nullptr, s.lam, nullptr, 2) == EIG33_ENOTSYM);
    CHECK(eig33cu_last_notsym_index() == (long long)(n - 3));
  }
  // several host threads driving the pipelines (and the shared copy pool) at once
  std::vector<std::thread> th;
  for (int t = 0; t < 4; ++t)
    th.emplace_back([t] {
      Batch b(5000 + 13 * t, false, false, 100 + t);
      for (int r = 0; r < 3; ++r) {
        CHECK(eig33_eigvals_host(b.a, b.n, b.inv, b.lam, b.fl, t & 1) == EIG33_OK);
        expect(b, 0, true, true);
      }
    });
  for (auto& x : th) x.join();
}

// MOCK_FAIL_LAUNCH_AT=k makes the k-th kernel launch fail: the call must
// return EIG33_ECUDA (never crash) and the next call must work.
static void fail() {
  const int fail_at = atoi(getenv("MOCK_FAIL_LAUNCH_AT") ? getenv("MOCK_FAIL_LAUNCH_AT") : "0");
  for (int pinned = 0; pinned < 2; ++pinned) {
    const size_t n = 5 * 1024 + 3;  // several chunks on either path
    Batch b(n, pinned, false, 7);
    mock_reset();
    const int rc = eig33_eigvals_host(b.a, n, b.inv, b.lam, b.fl, 0);
    if (fail_at >= 1 && mock_launches() >= fail_at) {
      CHECK(rc == EIG33_ECUDA);
      CHECK(strstr(eig33cu_last_error(), "mock launch failure") != nullptr);
    } else {
      CHECK(rc == EIG33_OK);
    }
    CHECK(eig33_eigvals_host(b.a, n, b.inv, b.lam, b.fl, 0) == EIG33_OK);
    expect(b, 0, true, true);
    mock_reset();
    const int rm = eig33_multi_eigvals(b.a, n, nullptr, b.lam, nullptr, 2);
    CHECK(rm == ((fail_at >= 1 && mock_launches() >= fail_at) ? EIG33_ECUDA : EIG33_OK));
    CHECK(eig33_multi_eigvals(b.a, n, nullptr, b.lam, nullptr, 2) == EIG33_OK);
    expect(b, 0, false, false);
  }
}

// the calling thread's current device survives host calls on other devices
static void device() {
  Batch b(5000, false, false, 3);
  for (int cur = 0; cur < 2; ++cur)
    for (int target = 0; target < 2; ++target) {
      CHECK(cudaSetDevice(cur) == cudaSuccess);
      CHECK(eig33_eigvals_host(b.a, b.n, nullptr, b.lam, nullptr, target) == EIG33_OK);
      int now = -1;
      cudaGetDevice(&now);
      CHECK(now == cur);
      CHECK(eig33_eigvals_host(b.a, b.n, nullptr, b.lam, nullptr, 7) == EIG33_EINVAL);
      cudaGetDevice(&now);
      CHECK(now == cur);
    }
}

int main(int argc, char** argv) {
  const std::string what = argc > 1 ? argv[1] : "basic";
  if (what == "basic") basic();
  if (what == "multi") multi();
  if (what == "fail") fail();
  if (what == "device") device();
  if (g_fail) {
    printf("FAILED %d\n", g_fail);
    return 1;
  }
  printf("OK %s\n", what.c_str());
  return 0;
}
