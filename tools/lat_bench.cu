// Dependent-chain latency of FP64 ops on the current GPU (one warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

template <int OP>
__global__ void chain(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  double x = seed + threadIdx.x * 1e-9;
  sm[threadIdx.x & 63] = x;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    if (OP == 0) x = __fma_rn(x, 0.999999, 1e-7);
    if (OP == 1) x = __dmul_rn(x, 1.0000001);
    if (OP == 2) x = rsqrt(x) + 0.5;
    if (OP == 3) x = sqrt(x) + 0.5;
    if (OP == 4) x = __drcp_rn(x) + 0.5;
    if (OP == 5) x = 1.0 / x + 0.5;
    if (OP == 6) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 0.9999999 + 1e-9;
    if (OP == 7) { sm[threadIdx.x & 63] = x; x = sm[(threadIdx.x + 1) & 63] * 0.9999999 + 1e-9; }
    if (OP == 8) x = (double)rsqrtf((float)x) + 0.5;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name) {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 256 * 8); cudaMalloc(&c, 8);
  chain<OP><<<1, 32>>>(d, c, 1.5);
  chain<OP><<<1, 32>>>(d, c, 1.5);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", name, (double)h / N);
  cudaFree(d); cudaFree(c);
}

int main() {
  run<0>("dfma");
  run<1>("dmul");
  run<2>("rsqrt+dadd");
  run<3>("sqrt+dadd");
  run<4>("drcp_rn+dadd");
  run<5>("ddiv+dadd");
  run<6>("shfl+dfma");
  run<7>("sts/lds+dfma");
  run<8>("rsqrtf(f32)+dadd");
  return 0;
}
