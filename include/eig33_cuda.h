/*
 * eig33_cuda.h -- C ABI of the B200 (sm_100a) batched eig33 hot path.
 *
 * Drop-in boundary for the reference's per-matrix C++ API
 * (/root/reference/proj/include/eig33/*.hpp), lifted to contiguous batches of
 * the same 72-byte row-major fp64 record (Mat3, include/eig33/mat3.hpp:24-28).
 * Plain pointers and sizes only; no exceptions cross it; every call returns a
 * status code:
 *   EIG33_OK (0), EIG33_ECUDA (1), EIG33_EINVAL (2), EIG33_ENOTSYM (3).
 * eig33cu_last_error() describes the last non-zero status of the calling thread.
 *
 * Device-pointer entry points (eig33cu_*) are stream-ordered and asynchronous
 * with respect to the host; `stream` is a cudaStream_t (NULL = legacy default
 * stream).  Host-pointer entry points (eig33_*_host, eig33_multi_*) are
 * synchronous and move data through pinned staging themselves.
 *
 * Packed output layouts (what the benchmark measures):
 *   inv   : n x 4 doubles {i1, j2, j3, disc}        (InvariantSet minus variant)
 *   lam   : n x 3 doubles {l1 <= l2 <= l3}          (EigenTriple minus the flag)
 *   flags : n bytes, bit0 = non_real_advisory, bit1 = not_symmetric (eigvalss)
 * Any of inv / flags may be NULL to skip that output.
 */
#ifndef EIG33_CUDA_H_
#define EIG33_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIG33_OK 0
#define EIG33_ECUDA 1
#define EIG33_EINVAL 2
#define EIG33_ENOTSYM 3

#define EIG33_FLAG_ADVISORY 0x1u
#define EIG33_FLAG_NOT_SYMMETRIC 0x2u

/* ABI version, (major << 16) | minor. */
int eig33cu_version(void);
/* Thread-local description of the last failure ("" if none). */
const char* eig33cu_last_error(void);
/* Thread-local: index (within the batch) of the first record that failed the
 * symmetry gate in the last eig33_eigvalss_host / eig33_multi_eigvalss call of
 * this thread, or -1.  The reference's scalar eigvalss throws NotSymmetric for
 * that record (src/eigensolver.cpp:102); the batch C++ wrapper rethrows it
 * with this index (include/eig33/batch.hpp). */
long long eig33cu_last_notsym_index(void);

/* Batched eig33::invariants(a, AlgorithmVariant::Stable)
 * (reference include/eig33/invariants.hpp:74, src/invariants.cpp:76-85).
 * Bit-exact.  d_a: n x 9 doubles, d_inv: n x 4 doubles. */
int eig33cu_invariants(const double* d_a, size_t n, double* d_inv, void* stream);

/* Batched eig33::eigvals (reference include/eig33/eigensolver.hpp:39,
 * src/eigensolver.cpp:91-95), fused with the invariants: they never
 * round-trip through HBM unless d_inv is non-NULL.  d_flags (optional)
 * receives non_real_advisory in bit0 (bit-exact vs src/eigensolver.cpp:54). */
int eig33cu_eigvals(const double* d_a, size_t n, double* d_inv, double* d_lam,
                    uint8_t* d_flags, void* stream);

/* Batched eig33::eigvalss (reference include/eig33/eigensolver.hpp:45,
 * src/eigensolver.cpp:97-117).  A matrix failing the symmetry gate (where the
 * scalar API throws NotSymmetric) gets NaN outputs and bit1 in d_flags. */
int eig33cu_eigvalss(const double* d_a, size_t n, double* d_inv, double* d_lam,
                     uint8_t* d_flags, void* stream);

/* Batched eig33::triple_angle (reference include/eig33/eigensolver.hpp:21,
 * src/eigensolver.cpp:84-89): phi[i] = atan2(sqrt(27*max(disc,0)), 27*j3). */
int eig33cu_triple_angle(const double* d_j3, const double* d_disc, size_t n, double* d_phi,
                         void* stream);

/* Accuracy-study variants (not on the throughput path), bit-exact like the rest:
 *  - eig33::invariants(a, v) for v = 0 Stable, 1 Naive, 2 NaiveTensor
 *    (reference include/eig33/invariants.hpp:74, src/invariants.cpp:76-98);
 *  - eig33::eigvals_naive (include/eig33/eigensolver.hpp:49, src/eigensolver.cpp:119-123),
 *    flags bit0 = non_real_advisory;
 *  - eig33::jacobian_j2 / jacobian_j3 / jacobian_disc (include/eig33/invariants.hpp:62-69,
 *    src/invariants.cpp:60-74): n x 9 row-major gradients, any output may be NULL. */
int eig33cu_invariants_variant(const double* d_a, size_t n, int variant, double* d_inv,
                               void* stream);
int eig33cu_eigvals_naive(const double* d_a, size_t n, double* d_lam, uint8_t* d_flags,
                          void* stream);
int eig33cu_jacobians(const double* d_a, size_t n, double* d_jj2, double* d_jj3, double* d_jdisc,
                      void* stream);
/* eig33::disc_naive(double j2, double j3) (include/eig33/invariants.hpp:59, src/invariants.cpp:58)
 * elementwise over n pairs: ((4 j2) j2) j2 - (27 j3) j3, bit-exact. */
int eig33cu_disc_naive(const double* d_j2, const double* d_j3, size_t n, double* d_disc,
                       void* stream);

/* Synchronous host-buffer versions on one device (chunked, pipelined
 * H2D / kernel / D2H over 3 streams; the calling thread's current device is
 * restored on return).  eig33_eigvalss_host returns EIG33_ENOTSYM if any
 * matrix failed the symmetry gate (outputs of all records still written;
 * eig33cu_last_notsym_index() names the first).  On an error return every
 * copy the call queued has completed: nothing writes caller memory later. */
int eig33_invariants_host(const double* h_a, size_t n, double* h_inv, int device);
/* invariants(a, variant) over host buffers, variant 0 Stable, 1 Naive, 2 NaiveTensor
 * (include/eig33/invariants.hpp:74, src/invariants.cpp:76-98). */
int eig33_invariants_variant_host(const double* h_a, size_t n, int variant, double* h_inv,
                                  int device);
int eig33_eigvals_host(const double* h_a, size_t n, double* h_inv, double* h_lam,
                       uint8_t* h_flags, int device);
int eig33_eigvalss_host(const double* h_a, size_t n, double* h_inv, double* h_lam,
                        uint8_t* h_flags, int device);

/* Multi-GPU host driver: contiguous even-aligned shards
 * [2*floor(g*n/(2G)), 2*floor((g+1)*n/(2G))) on devices 0..ngpu-1, one host
 * thread and stream set per device, no inter-GPU communication.  Results are
 * bitwise identical for every ngpu. */
int eig33_multi_eigvals(const double* h_a, size_t n, double* h_inv, double* h_lam,
                        uint8_t* h_flags, int ngpu);
/* Same, with an explicit device per shard: shard g (same bounds, G = ndev)
 * runs on devices[g]; a device may appear more than once. */
int eig33_multi_eigvals_on(const double* h_a, size_t n, double* h_inv, double* h_lam,
                           uint8_t* h_flags, const int* devices, int ndev);
int eig33_multi_invariants(const double* h_a, size_t n, double* h_inv, int ngpu);
int eig33_multi_eigvalss(const double* h_a, size_t n, double* h_inv, double* h_lam,
                         uint8_t* h_flags, int ngpu);

/* Synthetic corpora of the benchmark configs (BASELINE.json configs[0..4]),
 * counter-based: record i depends only on (config, seed, first_index + i), so
 * any shard regenerates independently.  config in 1..5. */
int eig33cu_generate(int config, uint64_t seed, uint64_t first_index, size_t n, double* d_a,
                     void* stream);

/* The paper's accuracy-sweep corpora: record i = generate_case(path, transform,
 * d_deltas[i]) = (U * diag(low, 1, 1 + delta)) * inverse_adjugate(U)
 * (reference include/eig33/bench.hpp:47, src/bench.cpp:53-75), bit-identical to
 * the reference.  path: 0 = D1, 1 = D2; kind: 0 = Symm, 1 = U1, 2 = U2 (gamma
 * must be nonzero, as make_transform requires). */
int eig33cu_generate_case(int path, int kind, double gamma, const double* d_deltas, size_t n,
                          double* d_a, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EIG33_CUDA_H_ */
