// Rank-b trailing update C -= Y X (K = b in {32, 64, 128}) fed by the Tensor
// Memory Accelerator: the second half of _block_stages (randomized.py:174-178),
// the roofline kernel of the RQRCP factorizations.
//
// One persistent CTA per SM -- its shared memory excludes a second CTA, so
// the pivot selection that runs beside it (driver.cu, select || trailing)
// keeps its SMs -- holding three independent groups of 4 warps.  Each group
// runs the TMA pipeline of tc_tma_kernel on its own 64 x 64 output tiles
// (tiles t_lo + g, t_lo + g + 3, ... of the CTA's contiguous range) with its
// own mbarriers and a named barrier, so one group's epilogue and pipeline
// fill overlap the others' DMMAs -- the effect of three small CTAs per SM
// (tc_gemm's best configuration) inside one exclusive CTA.  Y and X tiles
// are 64 x KG / KG x 64 boxes per stage (128-byte / 64-byte swizzles).  The
// default variant (ru_tma = 2: two stages of k 16) also fetches the group's
// 64 x 64 C tile by TMA when the tile starts, so the epilogue C - acc reads
// C from shared memory instead of waiting on HBM after the last DMMA
// (cfg2's K = 64 update 13.7 -> 15.8 TF/s beside the select, cfg5's K = 128
// 23.2 -> 25.2 TF/s; profiles/r02_ru_variants.jsonl).
#include "runtime.hpp"
#include "tc_tma.cuh"
#include "tma_util.hpp"

namespace rq {

namespace {

constexpr int kGM = 64, kGN = 64, kGroups = 3;
constexpr int kGThreads = kGroups * 128;
constexpr int kGCTile = kGM * kGN * 8;                       // 32 KB: one C tile

// KG: k per stage; STG: stages per group; CPRE: the group's C tile is fetched
// by TMA at the start of the tile into its own 32 KB buffer, so the epilogue
// reads C from shared memory instead of waiting on HBM after the last DMMA
template <int KG, int STG, bool CPRE>
struct GCfg {
  static constexpr int kStage = (kGM + kGN) * KG * 8;
  static constexpr int kGroupBytes = STG * kStage + (CPRE ? kGCTile : 0);
  static constexpr int kSmem = kGroups * kGroupBytes + 1024;
  static_assert(kSmem <= 227 * 1024, "one CTA per SM must fit");
};

struct RutArgs {
  int64_t M, N;
  int K;
  double* C; int64_t ldc;
  const Status* st;
  Status* snap;
};

RQ_DEV void group_sync(int gi) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "r"(128) : "memory");
}

// byte offset of Y(m, k) in a stage: boxes of 16 rows x KG k, rows k of 128
// bytes, 128-byte swizzle (chunk ^ (k & 7))
template <int KG>
RQ_DEV int off_y(int m, int k) {
  return (m >> 4) * (KG * 128) + k * 128 + (((((m & 15) >> 1) ^ k) & 7) << 4) + ((m & 1) << 3);
}
// byte offset of C(m, c) in the C tile: boxes of 16 rows x 64 columns, same swizzle
RQ_DEV int off_c(int m, int c) {
  return (m >> 4) * 8192 + c * 128 + (((((m & 15) >> 1) ^ c) & 7) << 4) + ((m & 1) << 3);
}

template <int KG, int STG, bool CPRE>
__global__ void __launch_bounds__(kGThreads, 1)
    rank_update_grouped_kernel(const __grid_constant__ CUtensorMap tmY,
                               const __grid_constant__ CUtensorMap tmX,
                               const __grid_constant__ CUtensorMap tmC, RutArgs a) {
  using Cfg = GCfg<KG, STG, CPRE>;
  if (a.snap != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    a.snap->abort = a.st != nullptr ? *((volatile const int*)&a.st->abort) : 0;
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) unsigned char ru_dsm[];
  unsigned char* base = ru_dsm + ((1024 - (smem_u32(ru_dsm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bars[kGroups][STG + 1];

  const int tid = threadIdx.x, gi = tid >> 7, gt = tid & 127;
  const int lane = gt & 31, warp = gt >> 5;
  const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t M = a.M, N = a.N, ldc = a.ldc;
  const int K = a.K, ktiles = K / KG;
  const int64_t tm = (M + kGM - 1) / kGM, tn = (N + kGN - 1) / kGN;
  const int64_t ntiles = tm * tn;
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  unsigned char* gbase = base + gi * Cfg::kGroupBytes;
  unsigned char* cbuf = gbase + STG * Cfg::kStage;   // CPRE only (1024-aligned)
  uint64_t* gbar = bars[gi];
  uint64_t* cbar = &bars[gi][STG];

  if (gt == 0) {
    for (int s = 0; s < STG + 1; ++s) mbar_init(&gbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int64_t it = 0;   // this group's running k-tile count (stage = it % S, parity = it / S)
  unsigned tpar = 0;  // parity of the C-tile barrier
  for (int64_t t = t_lo + gi; t < t_hi; t += kGroups) {
    // m fastest: consecutive tiles of a CTA share their X block in L2
    const int64_t m0 = (t % tm) * kGM, n0 = (t / tm) * kGN;
    auto issue = [&](int64_t j) {   // k-tile j of this tile, thread gt == 0
      const int s = (int)((it + j) % STG);
      unsigned char* st = gbase + s * Cfg::kStage;
      mbar_expect_tx(&gbar[s], Cfg::kStage);
#pragma unroll
      for (int b = 0; b < kGM / 16; ++b)
        tma_load_2d(st + b * (KG * 128), &tmY, (int)(m0 + 16 * b), (int)(j * KG), &gbar[s]);
#pragma unroll
      for (int b = 0; b < KG / 8; ++b)
        tma_load_2d(st + kGM * KG * 8 + b * (kGN * 64), &tmX, (int)(j * KG + 8 * b), (int)n0,
                    &gbar[s]);
    };
    group_sync(gi);   // the previous tile's stages (and C tile) are no longer read
    if (gt == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int j = 0; j < STG - 1 && j < ktiles; ++j) issue(j);
      if (CPRE) {
        mbar_expect_tx(cbar, kGCTile);
#pragma unroll
        for (int b = 0; b < kGM / 16; ++b)
          tma_load_2d(cbuf + b * 8192, &tmC, (int)(m0 + 16 * b), (int)n0, cbar);
      }
    }
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = (int)((it + kt) % STG);
      mbar_wait(&gbar[s], (unsigned)(((it + kt) / STG) & 1));
      group_sync(gi);   // stage (kt - 1) is free
      if (gt == 0 && kt + STG - 1 < ktiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(kt + STG - 1);
      }
      const unsigned char* sa = gbase + s * Cfg::kStage;
      const unsigned char* sb = sa + kGM * KG * 8;
#pragma unroll
      for (int k8 = 0; k8 < KG; k8 += 8) {
        double af[2][4], bf[2][4];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int m = wm0 + 16 * g + 2 * fr;
          const double2 v0 = *reinterpret_cast<const double2*>(sa + off_y<KG>(m, k8 + 2 * fk));
          const double2 v1 = *reinterpret_cast<const double2*>(sa + off_y<KG>(m, k8 + 2 * fk + 1));
          af[0][2 * g] = v0.x; af[0][2 * g + 1] = v0.y;
          af[1][2 * g] = v1.x; af[1][2 * g + 1] = v1.y;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double2 v =
              *reinterpret_cast<const double2*>(sb + tma_off_b<false, kGN>(wn0 + 8 * b + fr, k8 + 2 * fk));
          bf[0][b] = v.x; bf[1][b] = v.y;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) dmma884(acc[x][y], af[h][x], bf[h][y]);
      }
    }
    it += ktiles;
    // C - acc (numpy's C - Y @ X); rows 2g, 2g + 1 of a fragment pair are
    // consecutive: 16-byte loads and stores on full tiles
    const bool full = m0 + kGM <= M && n0 + kGN <= N;
    if (CPRE) {
      mbar_wait(cbar, tpar);
      tpar ^= 1u;
    }
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int rl = wm0 + 16 * g + 2 * fr;
      const int64_t r = m0 + rl;
      double2 cv[4][2];
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cl = wn0 + 8 * b + 2 * fk + e;
          const int64_t c = n0 + cl;
          if (CPRE) {   // out-of-range rows / columns were zero-filled by TMA
            cv[b][e] = *reinterpret_cast<const double2*>(cbuf + off_c(rl, cl));
          } else {
            const double* p = a.C + r + c * ldc;
            if (full) {
              cv[b][e] = __ldcs(reinterpret_cast<const double2*>(p));
            } else {
              cv[b][e].x = (r < M && c < N) ? p[0] : 0.0;
              cv[b][e].y = (r + 1 < M && c < N) ? p[1] : 0.0;
            }
          }
        }
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + wn0 + 8 * b + 2 * fk + e;
          double2 o;
          o.x = __dsub_rn(cv[b][e].x, acc[2 * g][b][e]);
          o.y = __dsub_rn(cv[b][e].y, acc[2 * g + 1][b][e]);
          double* p = a.C + r + c * ldc;
          if (full) {
            __stcg(reinterpret_cast<double2*>(p), o);
          } else if (c < N) {
            if (r < M) p[0] = o.x;
            if (r + 1 < M) p[1] = o.y;
          }
        }
    }
  }
}

template <int KG, int STG, bool CPRE>
void launch_grouped(int grid, const CUtensorMap& ty, const CUtensorMap& tx, const CUtensorMap& tc,
                    const RutArgs& a, cudaStream_t s) {
  using Cfg = GCfg<KG, STG, CPRE>;
  const void* fn = (const void*)rank_update_grouped_kernel<KG, STG, CPRE>;
  kernel_attr(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  rank_update_grouped_kernel<KG, STG, CPRE><<<grid, kGThreads, Cfg::kSmem, s>>>(ty, tx, tc, a);
}

}  // namespace

bool rank_update_tma(Handle& h, int64_t M, int64_t N, int64_t K, const double* Y, int64_t ldy,
                     const double* X, int64_t ldx, double* C, int64_t ldc, cudaStream_t s,
                     const Status* st, int cat, int max_ctas, Status* snap) {
  if (h.ru_tma <= 0 || (K != 32 && K != 64 && K != 128) || M < kGM || N <= 0) return false;
  const auto al = [](const void* p, int64_t ld) { return ((uintptr_t)p & 15) == 0 && ld % 2 == 0; };
  if (!al(Y, ldy) || !al(X, ldx) || !al(C, ldc)) return false;
  const int64_t tiles = ((M + kGM - 1) / kGM) * ((N + kGN - 1) / kGN);
  const int cap = max_ctas > 0 ? std::min(max_ctas, h.num_sms) : h.num_sms;
  const int grid = (int)std::min<int64_t>(cap, (tiles + kGroups - 1) / kGroups);
  ProfScope prof(h, cat, 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + 2.0 * M * N), s);
  // variant: 1 = 3 stages of k 16, C read from HBM in the epilogue; 2 = 2 stages
  // of k 16 + the C tile prefetched by TMA; 3 = 4 stages of k 8 + C prefetch
  const int v = h.ru_tma;
  const int kg = v == 3 ? 8 : 16;
  const CUtensorMap ty = tensor_map_f64(Y, M, K, ldy, 16, kg, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tx = tensor_map_f64(X, K, N, ldx, 8, kGN, CU_TENSOR_MAP_SWIZZLE_64B);
  const CUtensorMap tc = v >= 2 ? tensor_map_f64(C, M, N, ldc, 16, kGN, CU_TENSOR_MAP_SWIZZLE_128B) : tx;
  RutArgs a{M, N, (int)K, C, ldc, st, snap};
  if (v == 2) launch_grouped<16, 2, true>(grid, ty, tx, tc, a, s);
  else if (v == 3) launch_grouped<8, 4, true>(grid, ty, tx, tc, a, s);
  else launch_grouped<16, 3, false>(grid, ty, tx, tc, a, s);
  RQ_CHECK_LAUNCH();
  count_launch();
  return true;
}

}  // namespace rq
