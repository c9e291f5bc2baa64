// Tile-configuration sweep for the FP64 DMMA GEMMs (csrc/tc_gemm.cuh and the
// round-1 gemm_f64_kernel) on the hot path's product shapes, with cuBLAS as
// the yardstick (tool only; the library does not link cuBLAS for these).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1509_06820_b200/csrc -o tools/tc_sweep tools/tc_sweep.cu -lcublas
//   tools/tc_sweep            # JSON lines: shape, config, TF/s, occupancy, max error
#include <cublas_v2.h>

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "tc_gemm.cuh"
#include "tc_old.cuh"

using namespace rq;

namespace rq {
__global__ void gemm_reduce_kernel(GemmArgs g) {
  const int64_t total = g.M * g.N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double sum = g.partial[idx];
    for (int z = 1; z < g.splits; ++z) sum += g.partial[(size_t)z * total + idx];
    const int64_t r = idx % g.M, c = idx / g.M;
    g.C[r + c * g.ldc] = gemm_combine(sum, g.beta == 0.0 ? 0.0 : g.C[r + c * g.ldc], g.alpha, g.beta);
  }
}
}  // namespace rq

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

struct Shape {
  const char* name;
  bool ta, tb;
  int64_t M, N, K;
};

double* g_partial = nullptr;
double* g_ref = nullptr;
double* g_out = nullptr;
cublasHandle_t g_cub;

__global__ void init_kernel(double* p, int64_t n, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    p[i] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}
__global__ void maxdiff_kernel(const double* a, const double* b, int64_t n, double* out) {
  double m = 0, s = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    m = fmax(m, fabs(a[i] - b[i]));
    s = fmax(s, fabs(b[i]));
  }
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(~0u, m, o));
    s = fmax(s, __shfl_xor_sync(~0u, s, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax((unsigned long long*)out, __double_as_longlong(m));
    atomicMax((unsigned long long*)out + 1, __double_as_longlong(s));
  }
}

template <class Kern>
void run(const char* cfgname, Kern kern, int threads, size_t smem, int BM, int BN, int BK,
         const Shape& s, const double* A, const double* B, int reps, float cub_ms) {
  if (smem > 227 * 1024) return;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  GemmArgs g{};
  g.M = s.M; g.N = s.N; g.K = s.K;
  g.A = A; g.lda = s.ta ? s.K : s.M;
  g.B = B; g.ldb = s.tb ? s.N : s.K;
  g.C = g_out; g.ldc = s.M;
  g.alpha = 1.0; g.beta = 0.0;
  const int64_t gm = (s.M + BM - 1) / BM, gn = (s.N + BN - 1) / BN, tiles = gm * gn;
  const int64_t kt = (s.K + BK - 1) / BK;
  const int slots = 148 * (occ > 0 ? occ : 1);
  int best = 1;
  double bt = 1e300;
  for (int sp = 1; sp <= 32 && sp <= kt / 8 && (double)sp * s.M * s.N * 8 <= (1 << 30); ++sp) {
    const double waves = std::ceil((double)(tiles * sp) / slots);
    const double t = waves * (std::ceil((double)kt / sp) + 3.0) + (sp > 1 ? 0.02 * kt : 0);
    if (t < bt - 1e-9) { bt = t; best = sp; }
  }
  g.splits = best;
  const int64_t kc = (kt + best - 1) / best * BK;
  g.kchunk = best > 1 ? kc : s.K;
  g.splits = best > 1 ? (int)((s.K + kc - 1) / kc) : 1;
  g.partial = g_partial;
  const bool oned = std::string(cfgname).rfind("tc<", 0) == 0;
  auto launch = [&] {
    dim3 grid = oned ? dim3((unsigned)(gm * gn * g.splits)) : dim3((unsigned)gm, (unsigned)gn, (unsigned)g.splits);
    kern<<<grid, threads, smem>>>(g);
    if (g.splits > 1) gemm_reduce_kernel<<<148 * 8, 256>>>(g);
  };
  launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  double* d;
  CK(cudaMalloc(&d, 16));
  CK(cudaMemset(d, 0, 16));
  maxdiff_kernel<<<148 * 4, 256>>>(g_out, g_ref, s.M * s.N, d);
  double h[2];
  CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double tf = 2.0 * s.M * s.N * s.K / (ms * 1e-3) / 1e12;
  printf("{\"shape\": \"%s\", \"cfg\": \"%s\", \"tflops\": %.2f, \"cublas_tflops\": %.2f, "
         "\"occ\": %d, \"regs\": %d, \"smem\": %zu, \"splits\": %d, \"err\": %.2e}\n",
         s.name, cfgname, tf, 2.0 * s.M * s.N * s.K / (cub_ms * 1e-3) / 1e12, occ, fa.numRegs,
         smem, g.splits, h[0] / h[1]);
  fflush(stdout);
}

#define TC(TA, TB, BM, BN, BK, WM, WN, ST, MINB, DBUF)                                          \
  run("tc<" #BM "x" #BN "x" #BK ",w" #WM "x" #WN ",s" #ST ",minb" #MINB ",db" #DBUF ">",       \
      tc_gemm_kernel<TA, TB, BM, BN, BK, WM, WN, ST, 2, MINB, DBUF>,                            \
      TcCfg<TA, TB, BM, BN, BK, WM, WN, ST>::kThreads, TcCfg<TA, TB, BM, BN, BK, WM, WN, ST>::kSmem, \
      BM, BN, BK, s, A, B, reps, cub_ms)
#define TCO(TA, TB, BM, BN, BK, WM, WN, ST, MINB, DBUF)                                          \
  run("tcold<" #BM "x" #BN "x" #BK ",w" #WM "x" #WN ",s" #ST ",minb" #MINB ",db" #DBUF ">",       \
      tc_gemm_kernel_old<TA, TB, BM, BN, BK, WM, WN, ST, 2, MINB, DBUF>,                            \
      TcCfgOld<TA, TB, BM, BN, BK, WM, WN, ST>::kThreads, TcCfgOld<TA, TB, BM, BN, BK, WM, WN, ST>::kSmem, \
      BM, BN, BK, s, A, B, reps, cub_ms)
#define OLD(TA, TB, BM, BN, BK, WM, WN, ST)                                                      \
  run("old<" #BM "x" #BN "x" #BK ",w" #WM "x" #WN ",s" #ST ">",                                 \
      gemm_f64_kernel<TA, TB, BM, BN, BK, WM, WN, ST, 2>,                                        \
      GemmCfg<TA, TB, BM, BN, BK, WM, WN, ST>::kThreads, GemmCfg<TA, TB, BM, BN, BK, WM, WN, ST>::kSmem, \
      BM, BN, BK, s, A, B, reps, cub_ms)

template <bool TA, bool TB>
void sweep(const Shape& s, const double* A, const double* B, int reps, int which) {
  // cuBLAS reference + timing
  const double one = 1.0, zero = 0.0;
  auto cub = [&] {
    cublasDgemm(g_cub, TA ? CUBLAS_OP_T : CUBLAS_OP_N, TB ? CUBLAS_OP_T : CUBLAS_OP_N, (int)s.M,
                (int)s.N, (int)s.K, &one, A, (int)(TA ? s.K : s.M), B, (int)(TB ? s.N : s.K), &zero,
                g_ref, (int)s.M);
  };
  cub();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cub();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float cub_ms;
  cudaEventElapsedTime(&cub_ms, e0, e1);
  cub_ms /= reps;
  if (which == 0) {   // generic large
    TCO(TA, TB, 64, 64, 16, 32, 32, 3, 3, false);
    TC(TA, TB, 64, 64, 16, 32, 32, 3, 3, false);
    TC(TA, TB, 128, 64, 16, 64, 32, 3, 2, false);
  } else if (which == 2) {   // A^T with M = 32 (b = 32 inner products)
    TC(TA, TB, 32, 64, 16, 16, 32, 4, 4, false);
    TC(TA, TB, 32, 128, 16, 32, 32, 3, 3, false);
    TC(TA, TB, 32, 128, 16, 16, 64, 3, 3, false);
    TC(TA, TB, 32, 64, 16, 32, 16, 4, 5, false);
    TC(TA, TB, 32, 128, 32, 32, 32, 3, 2, false);
    TC(TA, TB, 32, 64, 32, 16, 32, 3, 4, false);
    TC(TA, TB, 64, 64, 16, 32, 32, 3, 3, false);
  } else {
    TC(TA, TB, 48, 64, 16, 16, 32, 4, 4, false);
    TC(TA, TB, 80, 64, 16, 16, 32, 3, 3, false);
  }
}

int main(int argc, char** argv) {
  const int reps = 5;
  cublasCreate(&g_cub);
  const size_t big = 32768ull * 32768ull + 4096 * 136;
  double *A, *B;
  CK(cudaMalloc(&A, 8 * (size_t)(32768 * 256)));
  CK(cudaMalloc(&B, 8 * big));
  CK(cudaMalloc(&g_ref, 8 * (size_t)8192 * 8192));
  CK(cudaMalloc(&g_out, 8 * (size_t)8192 * 8192));
  CK(cudaMalloc(&g_partial, (size_t)1 << 30));
  init_kernel<<<148 * 8, 256>>>(A, 32768 * 256, 1);
  init_kernel<<<148 * 8, 256>>>(B, big, 2);
  CK(cudaDeviceSynchronize());
  std::vector<Shape> sh = {
      {"square_8192", false, false, 8192, 8192, 8192},
      {"inner_b128_cfg5", true, false, 128, 32640, 32768},
      {"trq_G_cfg3", true, false, 64, 16320, 16384},
      {"trq_G_cfg4", true, false, 32, 11968, 20000},
      {"trq_G_cfg4_late", true, false, 32, 11776, 19800},
      {"tuxv_AV", false, false, 20000, 256, 12000},
      {"sketch_cfg3", false, false, 72, 16384, 16384},
      {"sketch_cfg5", false, false, 136, 32768, 32768},
  };
  for (auto& s : sh) {
    if (argc > 1 && std::string(argv[1]) != s.name) continue;
    // A operand small (skinny or TN M=128): A buffer; B big
    const double* a = A;
    const double* b = B;
    if (s.M == 8192 || s.M == 20000) { a = B; b = A; }   // tall A from the big buffer
    if (s.M == 8192) b = B + 8192ull * 8192;
    const int which = (s.M == 72 || s.M == 136) ? 1 : (s.M == 32 ? 2 : 0);
    if (s.ta && !s.tb) sweep<true, false>(s, a, b, reps, which);
    else sweep<false, false>(s, a, b, reps, which);
  }
  return 0;
}
