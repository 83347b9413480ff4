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
__global__ void dfma_kernel(float *out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 0.999, c = 1e-3;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void f2f_kernel(float *out, int iters) {  // cvt.f64.f32 (F2F) throughput
  float a[8];
  double acc[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i, acc[i] = 0.0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double d;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(a[i]));
      acc[i] += d;  // DADD, half the conversions' count of FP64 ops
      a[i] = __int_as_float(__float_as_int(a[i]) ^ 1);
    }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
// the ACCUM_F64 epilogue per entry: ex2 + (int re-bias | cvt) + DFMA
template <bool CVT>
__global__ void epi64_kernel(float *out, int iters) {
  float t[8];
  double acc[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) t[i] = -(threadIdx.x & 7) * 0.1f - i * 0.01f;
  const double z = 0.37;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float k;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(k) : "f"(t[i]));
      double kd;
      if (CVT) {
        asm volatile("cvt.f64.f32 %0, %1;" : "=d"(kd) : "f"(k));
      } else {
        const unsigned b = __float_as_uint(k);
        kd = __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
      }
      acc[i & 3] = fma(kd, z, acc[i & 3]);
      t[i] = t[i] - 1e-7f;
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc[0] + acc[1] + acc[2] + acc[3]);
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
  const double df = rate(dfma_kernel, 5000, 8, out, sms);
  const double cv = rate(f2f_kernel, 5000, 8, out, sms);
  const double ei = rate(epi64_kernel<false>, 5000, 8, out, sms);
  const double ec = rate(epi64_kernel<true>, 5000, 8, out, sms);
  const double u = sms * mhz * 1e6;
  printf("{\"sms\": %d, \"ffma_per_s\": %.4g, \"ffma_per_clk_sm\": %.1f, \"ex2_per_s\": %.4g, "
         "\"ex2_per_clk_sm\": %.2f, \"dfma_per_clk_sm\": %.2f, \"cvt_f64_f32_per_clk_sm\": %.2f, "
         "\"epi64_int_rebias_per_clk_sm\": %.2f, \"epi64_cvt_per_clk_sm\": %.2f, "
         "\"clock_mhz_assumed\": %.0f}\n",
         sms, f, f / u, e, e / u, df / u, cv / u, ei / u, ec / u, mhz);
  return 0;
}
