// L2 / HBM bandwidth probe (can an L2-resident k strip beat the two-pass
// product for d <= 190?).  A buffer of S bytes is read (LDG.128, streaming over the whole
// buffer, every SM) R times, and separately written then read back (the strip round trip:
// 4 B/entry store + 4 B/entry load).  S below the 126 MB L2 measures L2 bandwidth, above it
// HBM.  Prints bytes/s per configuration; CUDA-event timed, best of 5.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_bw l2_bw.cu && ./l2_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_kernel(const float4 *__restrict__ p, size_t n4, int reps, float *out) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldcg(p + i);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;  // keep the loads
}
__global__ void write_kernel(float4 *__restrict__ p, size_t n4, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
      p[i] = make_float4((float)r, 1.f, 2.f, 3.f);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t sizes_mb[] = {16, 32, 48, 64, 96, 4096};
  float4 *buf;
  float *out;
  cudaMalloc(&buf, (size_t)4096 << 20);
  cudaMalloc(&out, 16);
  cudaMemset(buf, 0, (size_t)4096 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t mb : sizes_mb) {
    const size_t bytes = mb << 20, n4 = bytes / 16;
    const int reps = mb >= 1024 ? 2 : (int)(4096 / mb);
    float best_r = 1e30f, best_w = 1e30f;
    for (int t = 0; t < 5; ++t) {
      float ms;
      read_kernel<<<sms * 4, 512>>>(buf, n4, 1, out);  // warm (L2-resident when it fits)
      cudaEventRecord(a);
      read_kernel<<<sms * 4, 512>>>(buf, n4, reps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best_r) best_r = ms;
      cudaEventRecord(a);
      write_kernel<<<sms * 4, 512>>>(buf, n4, reps);
      read_kernel<<<sms * 4, 512>>>(buf, n4, reps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best_w) best_w = ms;
    }
    const double rb = (double)bytes * reps;
    printf("{\"buffer_MB\": %zu, \"read_TBps\": %.2f, \"write_then_read_TBps\": %.2f}\n", mb,
           rb / (best_r * 1e-3) / 1e12, 2 * rb / (best_w * 1e-3) / 1e12);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
