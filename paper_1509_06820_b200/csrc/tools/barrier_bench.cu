// Grid-barrier latency microbenchmark (cooperative launch): fence+atomicAdd
// vs red.release + ld.acquire, at several CTA counts; and cluster barriers.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_fence(unsigned* c, unsigned& ep) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ep += 1; unsigned target = ep * gridDim.x;
    __threadfence(); atomicAdd(c, 1u);
    unsigned s; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(s) : "l"(c) : "memory"); } while (s < target);
  }
  __syncthreads();
}
__device__ __forceinline__ void bar_red(unsigned* c, unsigned& ep) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ep += 1; unsigned target = ep * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(c) : "memory");
    unsigned s; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(s) : "l"(c) : "memory"); } while (s < target);
  }
  __syncthreads();
}
__global__ void k_fence(unsigned* c, int n) { unsigned ep = 0; for (int i = 0; i < n; ++i) bar_fence(c, ep); }
__global__ void k_red(unsigned* c, int n) { unsigned ep = 0; for (int i = 0; i < n; ++i) bar_red(c, ep); }
__global__ void k_cg(int n) { auto g = cg::this_grid(); for (int i = 0; i < n; ++i) g.sync(); }
__global__ void __cluster_dims__(16, 1, 1) k_cluster16(int n) { auto cl = cg::this_cluster(); for (int i = 0; i < n; ++i) cl.sync(); }
__global__ void __cluster_dims__(8, 1, 1) k_cluster8(int n) { auto cl = cg::this_cluster(); for (int i = 0; i < n; ++i) cl.sync(); }

int main() {
  unsigned* c; cudaMalloc(&c, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 2000;
  int grids[] = {16, 32, 64, 148};
  for (int gi = 0; gi < 4; ++gi) {
    int g = grids[gi];
    for (int kind = 0; kind < 3; ++kind) {
      cudaMemset(c, 0, 64);
      int nn = n; void* args2[] = {&c, &nn}; void* args1[] = {&nn};
      void* fn = kind == 0 ? (void*)k_fence : kind == 1 ? (void*)k_red : (void*)k_cg;
      cudaLaunchCooperativeKernel(fn, g, 256, kind < 2 ? args2 : args1, 0, 0);
      cudaDeviceSynchronize();
      cudaMemset(c, 0, 64);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, g, 256, kind < 2 ? args2 : args1, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("{\"kind\": \"%s\", \"ctas\": %d, \"us_per_barrier\": %.3f}\n", kind == 0 ? "fence+atomic" : kind == 1 ? "red.release" : "cg.grid", g, ms * 1e3 / n);
    }
  }
  cudaFuncSetAttribute(k_cluster16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  k_cluster16<<<16, 256>>>(10); cudaDeviceSynchronize();
  cudaEventRecord(a); k_cluster16<<<16, 256>>>(n); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"kind\": \"cluster16\", \"us_per_barrier\": %.3f, \"err\": \"%s\"}\n", ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  cudaEventRecord(a); k_cluster8<<<8, 256>>>(n); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"kind\": \"cluster8\", \"us_per_barrier\": %.3f, \"err\": \"%s\"}\n", ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
