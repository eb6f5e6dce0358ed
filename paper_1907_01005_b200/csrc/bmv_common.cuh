// Shared helpers of libbmv: error state and device buffer management.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "bmv.h"

namespace bmv {

void set_error(const char* fmt, ...);

#define BMV_CUDA_TRY(expr)                                                    \
  do {                                                                        \
    cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      ::bmv::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                       __FILE__, __LINE__);                                   \
      return BMV_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

// every kernel launch is followed by BMV_CHECK_LAUNCH(): it also counts it
// (bmv_launch_count, used by bench.py's gpu_launches)
void count_launch();

#define BMV_CHECK_LAUNCH()                                                    \
  do {                                                                        \
    ::bmv::count_launch();                                                    \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) {                                                  \
      ::bmv::set_error("kernel launch failed: %s (%s:%d)",                    \
                       cudaGetErrorString(e_), __FILE__, __LINE__);           \
      return BMV_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

// Copy a host array into a fresh device allocation (nullptr for n == 0).
template <class T>
int upload(const T* host, int64_t n, T** dev) {
  *dev = nullptr;
  if (n <= 0) return BMV_OK;
  if (host == nullptr) {
    set_error("null host array of length %lld", (long long)n);
    return BMV_ERR_INVALID;
  }
  BMV_CUDA_TRY(cudaMalloc((void**)dev, sizeof(T) * (size_t)n));
  BMV_CUDA_TRY(cudaMemcpy(*dev, host, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice));
  return BMV_OK;
}

inline void release(void* p) {
  if (p) cudaFree(p);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

}  // namespace bmv
