// barrier_probe.cu -- cost of the synchronization primitives the persistent solver can
// use on B200: cooperative-groups grid.sync() over every SM, a hand-rolled sense-reversal
// grid barrier (one arrive atomic per CTA + acquire polling), and cluster.sync().
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_probe barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_grid(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// counter[0] = arrivals, counter[1] = generation
__device__ __forceinline__ void my_grid_sync(unsigned* counter, unsigned nblocks, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen;
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    if (prev == nblocks - 1) {
      counter[0] = 0;
      __threadfence();
      atomicExch(counter + 1, g + 1);
    } else {
      while (ld_acquire(counter + 1) == g) {
      }
    }
    gen = g + 1;
  }
  __syncthreads();
}

__global__ void k_mygrid(int iters, unsigned* counter, long long* out) {
  unsigned gen = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) my_grid_sync(counter, gridDim.x, gen);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster(int iters, long long* out) {
  cg::cluster_group c = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) c.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  unsigned* counter;
  cudaMalloc(&out, 64);
  cudaMalloc(&counter, 64);
  cudaMemset(counter, 0, 64);
  const int iters = 2000;
  long long h;
  for (int threads : {256, 512}) {
    void* args[] = {(void*)&iters, (void*)&out};
    cudaLaunchCooperativeKernel((void*)k_grid, sms, threads, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("cg grid.sync (%d CTAs x %d): %.0f cycles = %.2f us\n", sms, threads, (double)h / iters,
           (double)h / iters / 1965.0);
    cudaMemset(counter, 0, 64);
    void* args2[] = {(void*)&iters, (void*)&counter, (void*)&out};
    cudaLaunchCooperativeKernel((void*)k_mygrid, sms, threads, args2, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("custom grid barrier (%d CTAs x %d): %.0f cycles = %.2f us\n", sms, threads,
           (double)h / iters, (double)h / iters / 1965.0);
  }
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  k_cluster<<<16, 512>>>(iters, out);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("cluster.sync (16 CTAs x 512): %.0f cycles = %.2f us (%s)\n", (double)h / iters,
         (double)h / iters / 1965.0, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
