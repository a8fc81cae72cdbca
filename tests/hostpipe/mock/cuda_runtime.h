// Mock CUDA runtime -- TEST INFRASTRUCTURE (tests/test_hostpipe.py).
//
// Just enough of the runtime API for paper_2511_00292_b200/csrc/eig33_host.cpp
// to compile and run on a CPU: "device" memory is host memory tagged with the
// device that allocated it, every copy is bounds-checked against the
// allocations it touches, streams execute synchronously, and kernel launches
// (the eig33cu_* entry points, mock_device.cpp) check that their buffers
// belong to the calling thread's current device.  Failures can be injected.
#pragma once
#include <stddef.h>
#include <stdint.h>

typedef int cudaError_t;
enum { cudaSuccess = 0, cudaErrorInvalidValue = 1, cudaErrorMemoryAllocation = 2,
       cudaErrorInvalidDevice = 101, cudaErrorLaunchFailure = 719 };
typedef struct MockStream* cudaStream_t;
typedef struct MockEvent* cudaEvent_t;
enum cudaMemcpyKind { cudaMemcpyHostToDevice = 1, cudaMemcpyDeviceToHost = 2 };
enum cudaMemoryType { cudaMemoryTypeUnregistered = 0, cudaMemoryTypeHost = 1, cudaMemoryTypeDevice = 2 };
struct cudaPointerAttributes {
  cudaMemoryType type;
  int device;
};
#define cudaStreamNonBlocking 1u
#define cudaEventDisableTiming 2u
#define cudaHostAllocPortable 1u

const char* cudaGetErrorString(cudaError_t e);
cudaError_t cudaGetLastError(void);
cudaError_t cudaGetDevice(int* d);
cudaError_t cudaSetDevice(int d);
cudaError_t cudaGetDeviceCount(int* n);
cudaError_t cudaMalloc(void** p, size_t bytes);
template <class T>
inline cudaError_t cudaMalloc(T** p, size_t bytes) {
  return cudaMalloc(reinterpret_cast<void**>(p), bytes);
}
cudaError_t cudaFree(void* p);
cudaError_t cudaHostAlloc(void** p, size_t bytes, unsigned flags);
cudaError_t cudaFreeHost(void* p);
cudaError_t cudaStreamCreateWithFlags(cudaStream_t* s, unsigned flags);
cudaError_t cudaStreamSynchronize(cudaStream_t s);
cudaError_t cudaEventCreateWithFlags(cudaEvent_t* e, unsigned flags);
cudaError_t cudaEventRecord(cudaEvent_t e, cudaStream_t s);
cudaError_t cudaEventSynchronize(cudaEvent_t e);
cudaError_t cudaMemcpyAsync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s);
cudaError_t cudaPointerGetAttributes(cudaPointerAttributes* a, const void* p);
