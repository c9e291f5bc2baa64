// FP64 peak microbenchmark for the roofline denominator (MEASURED_PEAKS.json
// has no FP64 entry): DMMA.8x8x4 (mma.sync f64) and FFMA64 throughput over
// all SMs, timed with CUDA events.  Prints one JSON line.
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void ffma_loop(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double m = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double best_dmma = 0, best_ffma = 0;
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int blocks = sms * 2;
    dmma_loop<<<blocks, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * 8 * (double)iters * blocks * warps;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_dmma) best_dmma = tf;
    ffma_loop<<<blocks, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    ffma_loop<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ff = 2.0 * 8 * (double)iters * blocks * warps * 32;
    const double tf2 = ff / (ms * 1e-3) / 1e12;
    if (tf2 > best_ffma) best_ffma = tf2;
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"dmma_f64_tflops\": %.3f, \"ffma64_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d, "
         "\"err\": \"%s\"}\n",
         best_dmma, best_ffma, sms, clk, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
