// eig33_gen.cu -- on-device synthetic corpora for the five BASELINE configs.
//
// Counter-based: record i of config c with seed s depends only on (c, s, i),
// so every shard of a multi-GPU run regenerates its own slice and a parity
// test can regenerate any sub-range.  Similarity products use the reference's
// association (V*D)*V^-1 with V^-1 = inverse_adjugate(V)
// (proj/src/bench.cpp:69-75, proj/src/mat3.cpp:20-26,49-64), evaluated
// without contraction like the reference core.
//
//   1  symmetric: A = (Q*diag(l))*Q^T, Q Haar (Gram-Schmidt of a Gaussian,
//      R_ii > 0), l_i ~ U[-1,1]; upper triangle mirrored so A is bitwise symmetric
//   2  coalescing: A = (V*diag(1,1+e,1+2e))*V^-1, V Haar, e = 10^-u, u ~ U[1,15]
//   3  throughput: A = (V*diag(l))*V^-1, V_ij ~ N(0,1) rejected unless
//      cond_2(V) <= 1e3, l_i ~ U[-10,10]
//   4  ill-conditioned: V = (U*diag(1,s,s^2))*W^T, U,W Haar, s = 10^-t, t ~ U[1,4];
//      l = (1, 1+e, 2), e = 10^-u, u ~ U[0,12]
//   5  edge/scaling, quarter = (i >> 20) & 3 (contiguous 2^20 blocks):
//      q0 near-scalar c*I + d*E (c ~ U[-1,1], E_ij ~ N(0,1), d = 10^-u, u ~ U[8,16]);
//      q1 exact repeated/triple: (U1*diag(x,x,y))*U1^-1, x,y in Z/64, |x|,|y| <= 16,
//         half with y = x; q2 diagonal (N(0,1), a quarter with a repeated entry);
//      q3 G_ij ~ N(0,1) scaled by 2^k, k ~ U{-500..500}
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/eig33_cuda.h"
#include "eig33_internal.h"

namespace eig33b {
namespace gen {

struct M3 {
  double e[9];
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Stream of independent draws for one record.
struct Rng {
  uint64_t key;
  uint64_t ctr;
  __device__ Rng(uint64_t seed, int config, uint64_t idx, uint32_t attempt)
      : key(mix64(seed ^ mix64(((uint64_t)config << 56) ^ idx ^ ((uint64_t)attempt << 40)))),
        ctr(0) {}
  __device__ uint64_t next() { return mix64(key + 0x9e3779b97f4a7c15ull * (++ctr)); }
  __device__ double uniform() { return (double)(next() >> 11) * 0x1p-53; }  // [0,1)
  __device__ double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  __device__ double gauss() {
    const double u1 = ((double)(next() >> 11) + 0.5) * 0x1p-53;  // (0,1)
    const double u2 = uniform();
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
};

__device__ M3 matmul(const M3& a, const M3& b) {
  M3 c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c.e[3 * i + j] = (a.e[3 * i] * b.e[j] + a.e[3 * i + 1] * b.e[3 + j]) + a.e[3 * i + 2] * b.e[6 + j];
  return c;
}
__device__ M3 transpose(const M3& a) {
  return {{a.e[0], a.e[3], a.e[6], a.e[1], a.e[4], a.e[7], a.e[2], a.e[5], a.e[8]}};
}
__device__ M3 cofactor(const M3& a) {
  M3 c;
  c.e[0] = a.e[4] * a.e[8] - a.e[5] * a.e[7];
  c.e[1] = a.e[5] * a.e[6] - a.e[3] * a.e[8];
  c.e[2] = a.e[3] * a.e[7] - a.e[4] * a.e[6];
  c.e[3] = a.e[2] * a.e[7] - a.e[1] * a.e[8];
  c.e[4] = a.e[0] * a.e[8] - a.e[2] * a.e[6];
  c.e[5] = a.e[1] * a.e[6] - a.e[0] * a.e[7];
  c.e[6] = a.e[1] * a.e[5] - a.e[2] * a.e[4];
  c.e[7] = a.e[2] * a.e[3] - a.e[0] * a.e[5];
  c.e[8] = a.e[0] * a.e[4] - a.e[1] * a.e[3];
  return c;
}
__device__ double det(const M3& a) {
  return (a.e[0] * (a.e[4] * a.e[8] - a.e[5] * a.e[7]) - a.e[1] * (a.e[3] * a.e[8] - a.e[5] * a.e[6])) +
         a.e[2] * (a.e[3] * a.e[7] - a.e[4] * a.e[6]);
}
__device__ M3 inverse_adjugate(const M3& a) {
  const double d = det(a);
  const M3 adj = transpose(cofactor(a));
  M3 r;
  for (int k = 0; k < 9; ++k) r.e[k] = adj.e[k] / d;
  return r;
}
__device__ M3 diag(double a, double b, double c) { return {{a, 0, 0, 0, b, 0, 0, 0, c}}; }
__device__ M3 similar(const M3& v, const M3& d) { return matmul(matmul(v, d), inverse_adjugate(v)); }

// Haar-orthogonal Q: modified Gram-Schmidt on the columns of a Gaussian matrix
// (equivalent to QR with R_ii > 0).
__device__ M3 haar(Rng& r) {
  double c[3][3];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) c[j][i] = r.gauss();
  for (int j = 0; j < 3; ++j) {
    for (int k = 0; k < j; ++k) {
      const double p = c[j][0] * c[k][0] + c[j][1] * c[k][1] + c[j][2] * c[k][2];
      for (int i = 0; i < 3; ++i) c[j][i] -= p * c[k][i];
    }
    const double nrm = sqrt(c[j][0] * c[j][0] + c[j][1] * c[j][1] + c[j][2] * c[j][2]);
    for (int i = 0; i < 3; ++i) c[j][i] /= nrm;
  }
  M3 q;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) q.e[3 * i + j] = c[j][i];
  return q;
}

// cond_2(V) from the eigenvalues of the SPD Gram matrix V^T V (closed form).
__device__ double cond2(const M3& v) {
  const M3 g = matmul(transpose(v), v);
  const double m = (g.e[0] + g.e[4] + g.e[8]) / 3.0;
  const double b0 = g.e[0] - m, b4 = g.e[4] - m, b8 = g.e[8] - m;
  const double p2 = (b0 * b0 + b4 * b4 + b8 * b8 + 2.0 * (g.e[1] * g.e[1] + g.e[2] * g.e[2] + g.e[5] * g.e[5])) / 6.0;
  const double p = sqrt(p2);
  if (p == 0.0) return 1.0;
  const double detb = b0 * (b4 * b8 - g.e[5] * g.e[5]) - g.e[1] * (g.e[1] * b8 - g.e[5] * g.e[2]) +
                      g.e[2] * (g.e[1] * g.e[5] - b4 * g.e[2]);
  double rr = detb / (2.0 * p * p2);
  rr = fmin(1.0, fmax(-1.0, rr));
  const double phi = acos(rr) / 3.0;
  const double hi = m + 2.0 * p * cos(phi);
  const double lo = m + 2.0 * p * cos(phi + 2.0943951023931957);
  if (!(lo > 0.0)) return 1e300;
  return sqrt(hi / lo);
}

__device__ M3 make(int config, uint64_t seed, uint64_t idx) {
  if (config == 1) {
    Rng r(seed, 1, idx, 0);
    const M3 q = haar(r);
    const double l0 = r.uniform(-1, 1), l1 = r.uniform(-1, 1), l2 = r.uniform(-1, 1);
    M3 a = matmul(matmul(q, diag(l0, l1, l2)), transpose(q));
    a.e[3] = a.e[1];
    a.e[6] = a.e[2];
    a.e[7] = a.e[5];
    return a;
  }
  if (config == 2) {
    Rng r(seed, 2, idx, 0);
    const M3 v = haar(r);
    const double eps = exp10(-r.uniform(1, 15));
    return similar(v, diag(1.0, 1.0 + eps, 1.0 + 2.0 * eps));
  }
  if (config == 3) {
    for (uint32_t attempt = 0;; ++attempt) {
      Rng r(seed, 3, idx, attempt);
      M3 v;
      for (int k = 0; k < 9; ++k) v.e[k] = r.gauss();
      if (!(cond2(v) <= 1e3) && attempt < 64) continue;
      const double l0 = r.uniform(-10, 10), l1 = r.uniform(-10, 10), l2 = r.uniform(-10, 10);
      return similar(v, diag(l0, l1, l2));
    }
  }
  if (config == 4) {
    Rng r(seed, 4, idx, 0);
    const M3 u = haar(r), w = haar(r);
    const double s = exp10(-r.uniform(1, 4));
    const M3 v = matmul(matmul(u, diag(1.0, s, s * s)), transpose(w));
    const double eps = exp10(-r.uniform(0, 12));
    return similar(v, diag(1.0, 1.0 + eps, 2.0));
  }
  // config 5
  Rng r(seed, 5, idx, 0);
  const int quarter = (int)((idx >> 20) & 3);
  M3 a;
  if (quarter == 0) {
    const double c = r.uniform(-1, 1);
    const double dl = exp10(-r.uniform(8, 16));
    for (int k = 0; k < 9; ++k) a.e[k] = dl * r.gauss();
    a.e[0] += c;
    a.e[4] += c;
    a.e[8] += c;
  } else if (quarter == 1) {
    const M3 u1 = {{1, -1, 1, 1, 1, 1, -1, -1, 1}};
    const double x = (double)((int64_t)(r.next() % 2049) - 1024) / 64.0;
    double y = (double)((int64_t)(r.next() % 2049) - 1024) / 64.0;
    if (r.next() & 1) y = x;
    a = similar(u1, diag(x, x, y));
  } else if (quarter == 2) {
    const double d0 = r.gauss(), d1 = r.gauss();
    const double d2 = (r.next() & 3) == 0 ? d0 : r.gauss();
    a = diag(d0, d1, d2);
  } else {
    const int k = (int)(r.next() % 1001) - 500;
    for (int j = 0; j < 9; ++j) a.e[j] = ldexp(r.gauss(), k);
  }
  return a;
}

__global__ void k_generate(int config, uint64_t seed, uint64_t first, long long n, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const M3 a = make(config, seed, first + (uint64_t)i);
#pragma unroll
    for (int k = 0; k < 9; ++k) out[i * 9 + k] = a.e[k];
  }
}

}  // namespace gen
}  // namespace eig33b

extern "C" int eig33cu_generate(int config, uint64_t seed, uint64_t first_index, size_t n,
                                double* d_a, void* stream) {
  eig33b::set_error("");
  if (n == 0) return EIG33_OK;
  if (config < 1 || config > 5 || !d_a) {
    eig33b::set_error("eig33cu_generate: bad argument");
    return EIG33_EINVAL;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = (long long)((n + 255) / 256);
  const long long grid = blocks < 16LL * sms ? blocks : 16LL * sms;
  eig33b::gen::k_generate<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(config, seed, first_index,
                                                                          (long long)n, d_a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    eig33b::set_error(std::string("k_generate launch: ") + cudaGetErrorString(e));
    return EIG33_ECUDA;
  }
  return EIG33_OK;
}

// ---------------------------------------------------------------------------
// The paper's accuracy-sweep corpora: generate_case(path,
// transform, delta) = (U * diag(low, 1, 1 + delta)) * inverse_adjugate(U),
// reference proj/src/bench.cpp:53-75, one record per delta.
//   path: 0 = D1 (low = 1), 1 = D2 (low = -1)
//   kind: 0 = Symm, 1 = U1, 2 = U2(gamma)
// ---------------------------------------------------------------------------
namespace eig33b {
namespace gen {

__device__ M3 make_transform(int kind, double gamma) {
  const double q = 0x1.6a09e667f3bcdp-1;  // fl(sqrt 2)/2, bench.cpp:56
  if (kind == 0) return {{q, -0.5, 0.5, q, 0.5, -0.5, 0.0, q, q}};
  if (kind == 1) return {{1, -1, 1, 1, 1, 1, -1, -1, 1}};
  return {{1, 1, 1, 1, 0, 1, 2, 1, 2.0 + gamma}};
}

__global__ void k_generate_case(int path, int kind, double gamma, const double* __restrict__ deltas,
                                long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const M3 u = make_transform(kind, gamma);
    const double low = path == 0 ? 1.0 : -1.0;
    const M3 a = similar(u, diag(low, 1.0, 1.0 + deltas[i]));
#pragma unroll
    for (int k = 0; k < 9; ++k) out[i * 9 + k] = a.e[k];
  }
}

}  // namespace gen
}  // namespace eig33b

extern "C" int eig33cu_generate_case(int path, int kind, double gamma, const double* d_deltas,
                                     size_t n, double* d_a, void* stream) {
  eig33b::set_error("");
  if (n == 0) return EIG33_OK;
  if (path < 0 || path > 1 || kind < 0 || kind > 2 || !d_deltas || !d_a ||
      (kind == 2 && gamma == 0.0)) {
    eig33b::set_error("eig33cu_generate_case: bad argument (gamma must be nonzero for U2)");
    return EIG33_EINVAL;
  }
  const long long blocks = (long long)((n + 255) / 256);
  const unsigned grid = (unsigned)(blocks < 4096 ? blocks : 4096);
  eig33b::gen::k_generate_case<<<grid, 256, 0, (cudaStream_t)stream>>>(path, kind, gamma, d_deltas,
                                                                      (long long)n, d_a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    eig33b::set_error(std::string("k_generate_case launch: ") + cudaGetErrorString(e));
    return EIG33_ECUDA;
  }
  return EIG33_OK;
}
