// Pipe-rate microbenchmarks on the box (measure the FP32-FMA and MUFU.EX2
// peaks the roofline denominators assume): every thread runs independent dependency chains so
// the pipe, not latency, binds.  Prints ops/s for the whole GPU and the implied ops/clk/SM at
// the clock nvidia-smi reports during the run (pass it as argv[1] in MHz, or 1965).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float *out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float b = 0.999f, c = 1e-3f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ex2_kernel(float *out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -(threadIdx.x & 7) * 0.1f - i * 0.01f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
      a[i] = -y;  // keeps the argument in (-1, 0]
    }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename K>
double rate(K kern, int iters, double ops_per_thread_iter, float *out, int sms) {
  const int blocks = sms * 4, threads = 512;
  kern<<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ops_per_thread_iter * iters * (double)blocks * threads / (ms * 1e-3);
}
int main(int argc, char **argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  cudaMalloc(&out, sizeof(float) * sms * 4 * 512);
  const double f = rate(ffma_kernel, 20000, 8, out, sms);
  const double e = rate(ex2_kernel, 5000, 8, out, sms);
  printf("{\"sms\": %d, \"ffma_per_s\": %.4g, \"ffma_per_clk_sm\": %.1f, \"ex2_per_s\": %.4g, "
         "\"ex2_per_clk_sm\": %.2f, \"clock_mhz_assumed\": %.0f}\n",
         sms, f, f / (sms * mhz * 1e6), e, e / (sms * mhz * 1e6), mhz);
  return 0;
}
