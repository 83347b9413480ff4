#include <cstdio>
#include <cuda_runtime.h>
// DMMA throughput probe: independent accumulators, back-to-back MMAs.
template <int SHAPE>
__global__ void k(double *out, int iters) {
  double acc[8][8];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) acc[i][j] = threadIdx.x * 1e-9 + i + j;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-6;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a[t]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int S> void run(const char *name, int warps, double *out) {
  int iters = 2000;
  const double fma_per = S == 0 ? 256 : S == 1 ? 512 : S == 2 ? 1024 : 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k<S><<<sms, warps * 32>>>(out, 10);
  cudaEventRecord(e0);
  k<S><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * fma_per * 8 * iters * warps * sms;
  printf("%-10s warps/SM %2d  %.2f ms  %.1f TFLOP/s\n", name, warps, ms, flops / ms / 1e9);
}
int main() {
  double *out; cudaMalloc(&out, 148 * 1024 * 8);
  for (int w : {4, 8, 16}) {
    run<0>("m8n8k4", w, out); run<1>("m16n8k4", w, out); run<2>("m16n8k8", w, out); run<3>("m16n8k16", w, out);
  }
  return 0;
}
