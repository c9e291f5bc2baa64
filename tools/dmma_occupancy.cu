// DMMA.8x8x4 throughput vs warps per SM and independent accumulators per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void loop(double* out, int iters) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}
template <int NACC>
void run(int sms, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  for (int wps : {4, 8, 12, 16, 24, 32}) {
    const int iters = 4000;
    const int threads = wps * 32 > 1024 ? 1024 : wps * 32;
    const int blocks = sms * (wps * 32 / threads);
    loop<NACC><<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    loop<NACC><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 256 * NACC * (double)iters * blocks * (threads / 32) / (ms * 1e-3) / 1e12;
    printf("{\"acc\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", NACC, wps, tf);
  }
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  run<4>(sms, out, e0, e1);
  run<8>(sms, out, e0, e1);
  run<16>(sms, out, e0, e1);
  return 0;
}
