// l1_probe.cu -- does read-only data stay cached in an SM across a grid barrier?
// Pointer-chases 16 dependent loads through a per-CTA 16 KB slice right after each
// grid.sync() with three load flavours (ld.global.nc, ld.global.cg, plain ld.global) and
// prints the average latency per load. Also: the same chase with no barrier in between
// (warm L1), and a chase through a 64 MB array (L2/HBM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1_probe l1_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int MODE>
__device__ __forceinline__ int ldx(const int* p) {
  int v;
  if (MODE == 0) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  if (MODE == 1) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  if (MODE == 2) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int MODE, bool SYNC>
__global__ void k_chase(const int* __restrict__ next, int slice, int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  const int* base = next + (size_t)blockIdx.x * slice;
  long long tot = 0;
  int idx = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    if (SYNC) g.sync();
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < 16; ++k) idx = ldx<MODE>(base + idx);
    const long long t1 = clock64();
    tot += t1 - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot + (idx == -1);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int slice = 4096;  // ints per CTA (16 KB)
  int* h = new int[(size_t)sms * slice];
  for (int b = 0; b < sms; ++b)
    for (int i = 0; i < slice; ++i) h[(size_t)b * slice + i] = (i * 97 + 131) % slice;
  int* d;
  long long* out;
  cudaMalloc(&d, sizeof(int) * (size_t)sms * slice);
  cudaMalloc(&out, sizeof(long long) * sms);
  cudaMemcpy(d, h, sizeof(int) * (size_t)sms * slice, cudaMemcpyHostToDevice);
  long long* ho = new long long[sms];
  const int iters = 200;
  auto run = [&](void* fn, const char* name) {
    void* args[] = {(void*)&d, (void*)&slice, (void*)&iters, (void*)&out};
    cudaLaunchCooperativeKernel(fn, sms, 256, args, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(ho, out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int b = 0; b < sms; ++b) mean += ho[b];
    mean /= sms * (double)iters * 16;
    printf("%-34s %7.1f cycles/load (%s)\n", name, mean, cudaGetErrorString(e));
  };
  run((void*)k_chase<0, true>, "ld.global.nc after grid.sync");
  run((void*)k_chase<1, true>, "ld.global.cg after grid.sync");
  run((void*)k_chase<2, true>, "ld.global.ca after grid.sync");
  run((void*)k_chase<0, false>, "ld.global.nc, no barrier");
  run((void*)k_chase<1, false>, "ld.global.cg, no barrier");
  run((void*)k_chase<2, false>, "ld.global.ca, no barrier");
  return 0;
}
