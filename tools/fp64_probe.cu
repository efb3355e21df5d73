// fp64_probe.cu -- B200 FP64 pipe micro-measurements that size the solver and
// preselection design: DFMA throughput / latency, division and square-root latency,
// DMMA (fp64 tensor core) throughput. Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o fp64_probe fp64_probe.cu ; run on the GPU box.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fma_tput(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-7;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_fma_lat(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3;
  const double b = 1.0000001, c = 1e-7;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (a == 12345.0) out[0] = a;
}

__global__ void k_div_lat(double* out, int iters, long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-3;
  const double b = 1.0000001;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) a = b / a;
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (a == 12345.0) out[0] = a;
}

__global__ void k_sqrt_lat(double* out, int iters, long long* cyc) {
  double a = 2.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) a = sqrt(a) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (a == 12345.0) out[0] = a;
}

__global__ void k_dmma_tput(double* out, int iters) {
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  double v = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(v), "d"(v));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(v), "d"(v));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                 : "+d"(e0), "+d"(e1) : "d"(v), "d"(v));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                 : "+d"(f0), "+d"(f1) : "d"(v), "d"(v));
  }
  if (c0 + d0 + e0 + f0 + c1 + d1 + e1 + f1 == 12345.0) out[0] = c0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64);
  cudaMalloc(&cyc, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int iters = 4096;
  // throughput: sms * 8 CTAs * 256 threads * 8 chains * iters FMAs
  k_fma_tput<<<sms * 8, 256>>>(out, 16);
  cudaEventRecord(a);
  k_fma_tput<<<sms * 8, 256>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double fmas = (double)sms * 8 * 256 * 8 * iters;
  printf("DFMA throughput: %.2f TFLOP/s (%.1f FMA/clk/SM at 1.965 GHz)\n", 2 * fmas / ms / 1e9,
         fmas / (ms * 1e-3) / sms / 1.965e9);
  long long h;
  k_fma_lat<<<1, 32>>>(out, iters, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", (double)h / iters);
  k_div_lat<<<1, 32>>>(out, iters, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DDIV dependent latency: %.1f cycles\n", (double)h / iters);
  k_sqrt_lat<<<1, 32>>>(out, iters, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DSQRT(+add) dependent latency: %.1f cycles\n", (double)h / iters);
  k_dmma_tput<<<sms * 4, 128>>>(out, 16);
  cudaEventRecord(a);
  k_dmma_tput<<<sms * 4, 128>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double flops = (double)sms * 4 * 4 * 4 * iters * (8 * 8 * 4 * 2);
  printf("DMMA m8n8k4 throughput: %.2f TFLOP/s\n", flops / ms / 1e9);
  return 0;
}
