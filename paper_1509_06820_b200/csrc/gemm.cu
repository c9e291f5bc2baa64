// Host launcher + split-K reduction for the FP64 DMMA GEMM (gemm.cuh).
#include "gemm.cuh"
#include "runtime.hpp"

namespace rq {

__global__ void gemm_reduce_kernel(GemmArgs g) {
  if (aborted(g.st)) return;
  const int64_t total = g.M * g.N;
  const size_t plane = (size_t)total;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double sum = g.partial[idx];
    for (int z = 1; z < g.splits; ++z) sum = __dadd_rn(sum, g.partial[z * plane + idx]);
    const int64_t r = idx % g.M, c = idx / g.M;
    double* cp = g.C + r + c * g.ldc;
    const double old = g.beta == 0.0 ? 0.0 : *cp;
    *cp = gemm_combine(sum, old, g.alpha, g.beta);
  }
}

namespace {

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int ST, int VEC>
void launch_cfg(Handle& h, GemmArgs g, cudaStream_t s) {
  using Cfg = GemmCfg<TA, TB, BM, BN, BK, WM, WN, ST>;
  auto kern = gemm_f64_kernel<TA, TB, BM, BN, BK, WM, WN, ST, VEC>;
  kernel_attr((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  const int64_t gm = (g.M + BM - 1) / BM, gn = (g.N + BN - 1) / BN;
  const int64_t tiles = gm * gn;
  g.splits = 1;
  g.kchunk = g.K > 0 ? g.K : 1;
  const int64_t want_ctas = 3LL * h.num_sms;
  if (tiles < want_ctas && g.K >= 1024) {
    int64_t sp = (want_ctas + tiles - 1) / tiles;
    sp = std::min<int64_t>(sp, g.K / 256);
    // keep the partial planes bounded (256 MiB)
    const int64_t cap = (256LL << 20) / (8 * std::max<int64_t>(1, g.M * g.N));
    sp = std::min<int64_t>(sp, std::max<int64_t>(1, cap));
    if (sp > 1) {
      int64_t kc = (g.K + sp - 1) / sp;
      kc = (kc + BK - 1) / BK * BK;
      g.kchunk = kc;
      g.splits = (int)((g.K + kc - 1) / kc);
    }
  }
  if (g.splits > 1)
    g.partial = (double*)h.buf("gemm_partial", (size_t)g.splits * g.M * g.N * 8, s);
  dim3 grid((unsigned)gm, (unsigned)gn, (unsigned)g.splits);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, s>>>(g);
  RQ_CHECK_LAUNCH();
  count_launch();
  if (g.splits > 1) {
    const int64_t total = g.M * g.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * h.num_sms);
    gemm_reduce_kernel<<<blocks, 256, 0, s>>>(g);
    RQ_CHECK_LAUNCH();
    count_launch();
  }
}

template <bool TA, bool TB, int VEC>
void launch_v(Handle& h, const GemmArgs& g, cudaStream_t s) {
  const int64_t tiles128 = ((g.M + 127) / 128) * ((g.N + 63) / 64);
  if (g.M >= 128 && tiles128 >= 2LL * h.num_sms)
    launch_cfg<TA, TB, 128, 64, 16, 32, 32, 3, VEC>(h, g, s);
  else
    launch_cfg<TA, TB, 64, 64, 16, 32, 32, 3, VEC>(h, g, s);
}

// 16-byte copies need 16-byte aligned bases and even leading dimensions
bool aligned16(const double* p, int64_t ld) {
  return ((uintptr_t)p & 15) == 0 && (ld % 2) == 0;
}

template <bool TA, bool TB>
void launch_t(Handle& h, const GemmArgs& g, cudaStream_t s) {
  if (h.gemm_vec16 && aligned16(g.A, g.lda) && aligned16(g.B, g.ldb))
    launch_v<TA, TB, 2>(h, g, s);
  else
    launch_v<TA, TB, 1>(h, g, s);
}

}  // namespace

void gemm(Handle& h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
          const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
          int64_t ldc, cudaStream_t s, const Status* st, int cat) {
  if (M <= 0 || N <= 0) return;
  // rank-b trailing updates C -= Y X go to the persistent double-buffered kernel
  if (!ta && !tb && alpha == -1.0 && beta == 1.0 && M >= 64 && N >= 64 && h.use_rank_update &&
      rank_update(h, M, N, K, A, lda, B, ldb, C, ldc, s, st, cat))
    return;
  // tall-skinny inner products G = Y^T C (b = 64) go to the stream-K kernel
  if (ta && !tb && M == 64 && alpha == 1.0 && beta == 0.0 &&
      inner_gemm(h, M, N, K, A, lda, B, ldb, C, ldc, s, st, 0, cat))
    return;
  if (K > 0 && tc_gemm(h, ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s, st, cat))
    return;
  // algorithmic traffic: read A, B (+ C when beta != 0), write C
  const double bytes = 8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0.0 ? 2 : 1));
  ProfScope prof(h, cat, 2.0 * (double)M * N * K, bytes, s);
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
  g.alpha = alpha; g.beta = beta; g.st = st;
  if (K <= 0) {  // C = beta * C
    g.A = C; g.B = C;  // never dereferenced (no k tiles)
  }
  if (!ta && !tb) launch_t<false, false>(h, g, s);
  else if (!ta && tb) launch_t<false, true>(h, g, s);
  else if (ta && !tb) launch_t<true, false>(h, g, s);
  else launch_t<true, true>(h, g, s);
}

}  // namespace rq
