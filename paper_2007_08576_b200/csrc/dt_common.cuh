// dt_common.cuh -- error plumbing and small device utilities shared by the .cu files.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/deformtrack_b200.h"

namespace dt {

void set_error(const char* fmt, ...);

#define DT_CHECK_CUDA(expr)                                                           \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      ::dt::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                      __LINE__);                                                      \
      return DT_ERR_CUDA;                                                             \
    }                                                                                 \
  } while (0)

#define DT_CHECK_LAUNCH() DT_CHECK_CUDA(cudaGetLastError())

#define DT_REQUIRE(cond, code, ...)  \
  do {                               \
    if (!(cond)) {                   \
      ::dt::set_error(__VA_ARGS__);  \
      return (code);                 \
    }                                \
  } while (0)

// Device-side bounds checks of the checked build (-DDT_CHECKED, tools/checked_run.sh):
// every gather / scatter through an index that comes from another array (binding, CSR
// positions, edges, projected pixels, reduction slots) asserts its range and traps on a
// violation. compute-sanitizer is not available on this GPU pool, so this build plus the
// parity suite is the out-of-bounds evidence. Compiled out otherwise.
#ifdef DT_CHECKED
#define DT_DCHECK(cond)                                                                      \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("DT_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define DT_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 1 << 30) g = 1 << 30;
  return (int)g;
}

// Deterministic per-warp sum of NV doubles held per lane: each lane writes its NV
// partials to shared scratch (32 x NV), then lane c < NV sums the 32 partials of column c
// in lane order. The result lands in out[c] (shared or global) written by lane c.
template <int NV>
__device__ __forceinline__ void warp_column_sum(const double* vals, double* scratch, double* out) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < NV; ++c) scratch[lane * NV + c] = vals[c];
  __syncwarp();
  if (lane < NV) {
    double s = 0.0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) s += scratch[l * NV + lane];
    out[lane] = s;
  }
  __syncwarp();
}

// Deterministic warp reduction for a single double (fixed xor-tree order).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace dt
