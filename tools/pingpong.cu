// One-way signalling latency between two CTAs: DSMEM (cluster) vs L2 (grid),
// with the variants the select exchange can use.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pp tools/pingpong.cu && /tmp/pp
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int kIters = 2000;

__global__ void __cluster_dims__(2, 1, 1) pp_dsmem(long long* out, int mode) {
  __shared__ volatile unsigned long long box;
  auto cl = cg::this_cluster();
  const int me = cl.block_rank();
  if (threadIdx.x == 0) box = 0;
  cl.sync();
  if (threadIdx.x == 0) {
    volatile unsigned long long* peer = cl.map_shared_rank((unsigned long long*)&box, me ^ 1);
    long long t0 = clock64();
    for (int i = 1; i <= kIters; ++i) {
      if (me == 0) {
        if (mode == 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
        *peer = (unsigned long long)i;
        while (box != (unsigned long long)i) {}
      } else {
        while (box != (unsigned long long)i) {}
        if (mode == 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
        *peer = (unsigned long long)i;
      }
    }
    if (me == 0) out[0] = (clock64() - t0) / (2 * kIters);
  }
  cl.sync();
}

__global__ void pp_global(unsigned long long* box, long long* out, int mode) {
  const int me = blockIdx.x;
  if (threadIdx.x == 0) {
    unsigned long long* mine = box + 32 * me;
    unsigned long long* peer = box + 32 * (me ^ 1);
    long long t0 = clock64();
    for (int i = 1; i <= kIters; ++i) {
      auto wait = [&]() {
        unsigned long long v;
        do {
          if (mode == 2)
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
          else
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        } while (v != (unsigned long long)i);
      };
      auto send = [&]() {
        if (mode == 1) __threadfence();
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(peer), "l"((unsigned long long)i) : "memory");
      };
      if (me == 0) { send(); wait(); } else { wait(); send(); }
    }
    if (me == 0) out[0] = (clock64() - t0) / (2 * kIters);
  }
}

// fence cost with outstanding global stores
__global__ void fence_cost(double* buf, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < 100; ++i) {
    buf[threadIdx.x + 32 * i] = i;
    __threadfence();
  }
  if (threadIdx.x == 0) out[0] = (clock64() - t0) / 100;
}

int main() {
  long long *d, h;
  unsigned long long* box;
  double* buf;
  cudaMalloc(&d, 8);
  cudaMalloc(&box, 4096);
  cudaMalloc(&buf, 1 << 20);
  for (int mode = 0; mode < 2; ++mode) {
    pp_dsmem<<<2, 32>>>(d, mode);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"kind\": \"dsmem\", \"fence\": %d, \"one_way_cycles\": %lld}\n", mode, h);
  }
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(box, 0, 4096);
    pp_global<<<2, 32>>>(box, d, mode);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"kind\": \"global\", \"mode\": %d, \"one_way_cycles\": %lld}\n", mode, h);
  }
  fence_cost<<<1, 32>>>(buf, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"kind\": \"store+threadfence\", \"cycles\": %lld}\n", h);
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
