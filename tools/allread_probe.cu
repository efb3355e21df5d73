// allread_probe.cu -- cost of the "every CTA reads every item value after the grid
// barrier" pattern the LM solver uses for its cost totals: 148 CTAs x 512 threads, each
// CTA writes its slice of an N-double array, grid.sync(), then every CTA sums the whole
// array (4 loads in flight per thread, block reduce). Reports the mean per-CTA time from
// barrier release to total, per N; plus one-warp-per-CTA reading.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o allread_probe allread_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ long long gt() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool ONE_WARP>
__global__ void k_allread(double* vals, int n, int iters, long long* out, double* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ double s_part[16];
  long long tot = 0;
  double keep = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      vals[i] = i * 1e-3 + it;
    g.sync();
    const long long t0 = gt();
    double acc = 0;
    if (!ONE_WARP || threadIdx.x < 32) {
      const int stride = ONE_WARP ? 32 : blockDim.x;
      for (int i = threadIdx.x; i < n; i += stride) acc += __ldcg(vals + i);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    }
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    double t = 0;
    for (int w = 0; w < (ONE_WARP ? 1 : (int)blockDim.x / 32); ++w) t += s_part[w];
    keep += t;
    const long long t1 = gt();
    tot += t1 - t0;
    g.sync();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot;
  if (keep == 12345.0) sink[0] = keep;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* vals;
  double* sink;
  long long* out;
  cudaMalloc(&vals, 8 << 20);
  cudaMalloc(&sink, 64);
  cudaMalloc(&out, 8 * sms);
  long long* h = new long long[sms];
  const int iters = 200;
  for (int one = 0; one < 2; ++one)
    for (int n : {64, 256, 1024, 2048, 4096}) {
      void* args[] = {(void*)&vals, (void*)&n, (void*)&iters, (void*)&out, (void*)&sink};
      cudaLaunchCooperativeKernel(one ? (void*)k_allread<true> : (void*)k_allread<false>, sms, 512,
                                  args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, out, 8 * sms, cudaMemcpyDeviceToHost);
      double mean = 0, mx = 0;
      for (int b = 0; b < sms; ++b) {
        mean += h[b];
        mx = h[b] > mx ? h[b] : mx;
      }
      printf("%s n=%5d: mean %.2f us, max-CTA %.2f us (%s)\n", one ? "one warp " : "all warps", n,
             mean / sms / iters / 1e3, mx / iters / 1e3, cudaGetErrorString(e));
    }
  return 0;
}
