// Host launcher for the second-generation DMMA GEMM (tc_gemm.cuh): tile
// family choice by shape, split-K for grids that cannot fill the SMs
// (wave-quantisation aware), deterministic fixed-order reduction.
#include <algorithm>
#include <cmath>

#include "runtime.hpp"
#include "tc_gemm.cuh"
#include "tc_tma.cuh"
#include "tma_util.hpp"

namespace rq {

namespace {

// K chunks per output tile: maximise the occupied fraction of the last wave
// (one CTA per SM), each chunk at least `min_kt` k-tiles deep
int choose_splits(int64_t tiles, int64_t ktiles, int sms, int min_kt, int64_t plane,
                  int forced) {
  if (forced > 0) return (int)std::min<int64_t>(forced, std::max<int64_t>(1, ktiles));
  if (tiles >= 4LL * sms) return 1;
  const int64_t cap_mem = std::max<int64_t>(1, (512LL << 20) / (8 * std::max<int64_t>(1, plane)));
  const int64_t maxsp = std::min<int64_t>(std::min<int64_t>(32, std::max<int64_t>(1, ktiles / min_kt)), cap_mem);
  int best = 1;
  double best_t = 1e300;
  for (int64_t sp = 1; sp <= maxsp; ++sp) {
    const int64_t ctas = tiles * sp;
    const double waves = std::ceil((double)ctas / sms);
    // time ~ waves x (k-tiles per chunk + fill/epilogue overhead ~ 3 k-tiles)
    const double per = std::ceil((double)ktiles / sp) + 3.0;
    const double t = waves * per + (sp > 1 ? 0.02 * ktiles : 0.0);
    if (t < best_t - 1e-9) {
      best_t = t;
      best = (int)sp;
    }
  }
  return best;
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int ST, int VEC, int MINB,
          bool DBUF>
void tc_launch(Handle& h, GemmArgs g, cudaStream_t s, int forced_splits) {
  using Cfg = TcCfg<TA, TB, BM, BN, BK, WM, WN, ST>;
  auto kern = tc_gemm_kernel<TA, TB, BM, BN, BK, WM, WN, ST, VEC, MINB, DBUF>;
  kernel_attr((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
  const int64_t gm = (g.M + BM - 1) / BM, gn = (g.N + BN - 1) / BN;
  const int64_t ktiles = (g.K + BK - 1) / BK;
  // resident CTAs per SM: the launch bound's minimum (registers and shared
  // memory are sized for it)
  const int slots = h.num_sms * MINB;
  const int sp = g.K > 0 ? choose_splits(gm * gn, ktiles, slots, 8, g.M * g.N, forced_splits) : 1;
  g.splits = 1;
  g.kchunk = g.K > 0 ? g.K : 1;
  if (sp > 1) {
    const int64_t kc = (ktiles + sp - 1) / sp * BK;
    g.kchunk = kc;
    g.splits = (int)((g.K + kc - 1) / kc);
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

// Tile families (variant ids for the `tc_variant` option), chosen from a
// sweep against cuBLAS on the hot path's shapes (tools/tc_sweep.cu,
// profiles/r02_tc_sweep.jsonl).  Several small CTAs per SM beat one large
// one: a CTA's barrier and epilogue stalls are covered by its neighbours.
//   0   64 x  64 x 16, 4 warps of 32 x 32, 3 stages, 3 CTAs/SM   general
//   1  128 x  64 x 16, 4 warps of 64 x 32, 3 stages, 2 CTAs/SM   A^T with 64 < M (G = Y^T C, b = 128)
//   2   48 x  64 x 16, 6 warps of 16 x 32, 4 stages, 4 CTAs/SM   M <= 48, or 80 < M <= 144 (sketch l = 136)
//   3   80 x  64 x 16, 10 warps of 16 x 32, 3 stages, 3 CTAs/SM  64 < M <= 80 (sketch at l = 72)
//   4   32 x  64 x 16, 4 warps of 16 x 32, 4 stages, 4 CTAs/SM   A^T with M <= 32 (b = 32)
//   5   64 x 128 x 16, 4 warps of 32 x 64, 3 stages, 2 CTAs/SM   (cuBLAS-like; kept for sweeps)
template <bool TA, bool TB, int VEC>
void tc_dispatch(Handle& h, const GemmArgs& g, cudaStream_t s, int v, int sp) {
  switch (v) {
    case 1: tc_launch<TA, TB, 128, 64, 16, 64, 32, 3, VEC, 2, false>(h, g, s, sp); break;
    case 2: tc_launch<TA, TB, 48, 64, 16, 16, 32, 4, VEC, 4, false>(h, g, s, sp); break;
    case 3: tc_launch<TA, TB, 80, 64, 16, 16, 32, 3, VEC, 3, false>(h, g, s, sp); break;
    case 4: tc_launch<TA, TB, 32, 64, 16, 16, 32, 4, VEC, 4, false>(h, g, s, sp); break;
    case 5: tc_launch<TA, TB, 64, 128, 16, 32, 64, 3, VEC, 2, false>(h, g, s, sp); break;
    default: tc_launch<TA, TB, 64, 64, 16, 32, 32, 3, VEC, 3, false>(h, g, s, sp); break;
  }
}

int tc_pick(const Handle& h, bool ta, int64_t M) {
  if (h.tc_variant >= 0) return h.tc_variant;
  if (ta) {
    if (M <= 32) return 4;
    return M <= 64 ? 0 : 1;
  }
  if (M <= 48) return 2;
  if (M <= 64) return 0;
  if (M <= 80) return 3;
  if (M <= 144) return 2;
  return 0;
}

// ---- TMA-fed variants (tc_tma.cuh); tensor maps from tma_util.hpp
template <bool TA, bool TB, int BM, int BN, int WM, int WN, int ST, int MINB>
void tma_launch(Handle& h, GemmArgs g, cudaStream_t s, int forced_splits) {
  using Cfg = TmaCfg<TA, TB, BM, BN, WM, WN>;
  auto kern = tc_tma_kernel<TA, TB, BM, BN, WM, WN, ST, MINB>;
  constexpr size_t smem = (size_t)ST * Cfg::kStage + 1024;
  kernel_attr((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const CUtensorMap ta = TA ? tensor_map_f64(g.A, g.K, g.M, g.lda, 8, BM, CU_TENSOR_MAP_SWIZZLE_64B)
                            : tensor_map_f64(g.A, g.M, g.K, g.lda, 16, 16, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tb = TB ? tensor_map_f64(g.B, g.N, g.K, g.ldb, 16, 16, CU_TENSOR_MAP_SWIZZLE_128B)
                            : tensor_map_f64(g.B, g.K, g.N, g.ldb, 8, BN, CU_TENSOR_MAP_SWIZZLE_64B);
  const int64_t gm = (g.M + BM - 1) / BM, gn = (g.N + BN - 1) / BN;
  const int64_t ktiles = (g.K + Cfg::BK - 1) / Cfg::BK;
  const int sp = choose_splits(gm * gn, ktiles, h.num_sms * MINB, 8, g.M * g.N, forced_splits);
  g.splits = 1;
  g.kchunk = g.K;
  if (sp > 1) {
    const int64_t kc = (ktiles + sp - 1) / sp * Cfg::BK;
    g.kchunk = kc;
    g.splits = (int)((g.K + kc - 1) / kc);
  }
  if (g.splits > 1)
    g.partial = (double*)h.buf("gemm_partial", (size_t)g.splits * g.M * g.N * 8, s);
  dim3 grid((unsigned)gm, (unsigned)gn, (unsigned)g.splits);
  kern<<<grid, Cfg::kThreads, smem, s>>>(ta, tb, g);
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

template <bool TA, bool TB>
void tma_dispatch(Handle& h, const GemmArgs& g, cudaStream_t s, int v, int sp) {
  switch (v) {
    case 1: tma_launch<TA, TB, 128, 64, 64, 32, 3, 2>(h, g, s, sp); break;
    case 2: tma_launch<TA, TB, 48, 64, 16, 32, 4, 4>(h, g, s, sp); break;
    case 3: tma_launch<TA, TB, 80, 64, 16, 32, 3, 3>(h, g, s, sp); break;
    case 4: tma_launch<TA, TB, 32, 64, 16, 32, 4, 4>(h, g, s, sp); break;
    case 5: tma_launch<TA, TB, 64, 128, 32, 64, 3, 2>(h, g, s, sp); break;
    default: tma_launch<TA, TB, 64, 64, 32, 32, 3, 3>(h, g, s, sp); break;
  }
}

bool aligned16(const double* p, int64_t ld) { return ((uintptr_t)p & 15) == 0 && (ld % 2) == 0; }

}  // namespace

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    RQ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2-d tensor map of a column-major FP64 matrix: `inner` contiguous rows,
// `outer` columns, leading dimension ld; box inner x outer, swizzled
CUtensorMap tensor_map_f64(const double* base, int64_t inner, int64_t outer, int64_t ld, int box_in,
                       int box_out, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_in, (cuuint32_t)box_out};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims,
                                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
  return m;
}

bool tc_gemm(Handle& h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
             const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
             int64_t ldc, cudaStream_t s, const Status* st, int cat) {
  if (!h.use_tc || (ta && tb) || M <= 0 || N <= 0 || K <= 0) return false;
  const double bytes =
      8.0 * ((double)M * K + (double)K * N + (double)M * N * (beta != 0.0 ? 2 : 1));
  ProfScope prof(h, cat, 2.0 * (double)M * N * K, bytes, s);
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
  g.alpha = alpha; g.beta = beta; g.st = st;
  const int v = tc_pick(h, ta, M);
  const int sp = h.tc_splits;
  const bool vec = h.gemm_vec16 && aligned16(A, lda) && aligned16(B, ldb);
  if (h.tc_tma && vec) {
    if (ta) tma_dispatch<true, false>(h, g, s, v, sp);
    else if (tb) tma_dispatch<false, true>(h, g, s, v, sp);
    else tma_dispatch<false, false>(h, g, s, v, sp);
    return true;
  }
  if (!ta && !tb) {
    if (vec) tc_dispatch<false, false, 2>(h, g, s, v, sp);
    else tc_dispatch<false, false, 1>(h, g, s, v, sp);
  } else if (ta) {
    if (vec) tc_dispatch<true, false, 2>(h, g, s, v, sp);
    else tc_dispatch<true, false, 1>(h, g, s, v, sp);
  } else {
    if (vec) tc_dispatch<false, true, 2>(h, g, s, v, sp);
    else tc_dispatch<false, true, 1>(h, g, s, v, sp);
  }
  return true;
}

}  // namespace rq
