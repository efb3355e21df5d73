// dmma_probe.cu -- latency of the solver's FP64 building blocks on one warp:
// a dependent chain of DMMA.8x8x4 (same accumulator), one "Gram push" (32 rows x 8
// columns staged through shared memory, 8 DMMAs), a dependent DFMA chain, DDIV, DSQRT.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void k_probe(long long* out, double* sink) {
  __shared__ double stage[32 * 9];
  const int lane = threadIdx.x & 31;
  double c0 = 0, c1 = 0, v = lane * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) dmma884(c0, c1, v, v);
  long long t1 = clock64();
  out[0] = (t1 - t0) / 256;
  // gram push: stage a row, 8 dmma over the staged columns
  double row[8];
  for (int c = 0; c < 8; ++c) row[c] = lane + c;
  t0 = clock64();
  for (int it = 0; it < 64; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) stage[lane * 9 + c] = row[c] + c0 * 1e-300;
    __syncwarp();
    const int t = lane & 3, g = lane >> 2;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double x = stage[(4 * q + t) * 9 + g];
      dmma884(c0, c1, x, x);
    }
    __syncwarp();
  }
  t1 = clock64();
  out[1] = (t1 - t0) / 64;
  double a = v;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) a = fma(a, 1.0000001, 1e-9);
  t1 = clock64();
  out[2] = (t1 - t0) / 256;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) a = 1.0000001 / a;
  t1 = clock64();
  out[3] = (t1 - t0) / 256;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) a = sqrt(a) + 0.5;
  t1 = clock64();
  out[4] = (t1 - t0) / 256;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) a = acos(a * 1e-3);
  t1 = clock64();
  out[5] = (t1 - t0) / 256;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) a = sin(a) + 0.1;
  t1 = clock64();
  out[6] = (t1 - t0) / 256;
  sink[threadIdx.x] = c0 + c1 + a;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 64 * 8);
  cudaMalloc(&s, 64 * 8);
  k_probe<<<1, 32>>>(d, s);
  long long h[8];
  cudaMemcpy(h, d, 7 * 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency       %lld cycles\n", h[0]);
  printf("Gram push (stage + 8 DMMA)   %lld cycles\n", h[1]);
  printf("DFMA dependent latency       %lld cycles\n", h[2]);
  printf("DDIV dependent latency       %lld cycles\n", h[3]);
  printf("DSQRT+add dependent latency  %lld cycles\n", h[4]);
  printf("acos dependent latency       %lld cycles\n", h[5]);
  printf("sin+add dependent latency    %lld cycles\n", h[6]);
  return 0;
}
