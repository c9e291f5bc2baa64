// FP64 DMMA GEMM, second generation: C = alpha * op(A) op(B) + beta * C
// (column-major, explicit leading dimensions), for every plain product of the
// hot path that round 1 sent to cuBLAS:
//   sketch        B = Omega A                    (randomized.py:76; truncated.py:59, 63)
//   inner         G = Y^T C                      (randomized.py:172; truncated.py:144)
//   TUXV          A V, U^T A                     (truncated.py:230, 238)
//   blocked QR    apply_block_reflection         (kernels.py:166-181; qrcp.py:222-252)
//   dense Q       q_columns                      (qrcp.py:53-60)
//
// sm_100a has no FP64 tcgen05 kind, so the tensor instruction is the warp
// `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4).  What separates this kernel from
// gemm_f64_kernel (gemm.cuh) is how fragments reach the DMMA:
//
//  * k-pairs.  One 8-deep k step is two DMMAs; lane (fr, fk) supplies k =
//    2fk for the first and 2fk + 1 for the second (the 4 lanes of a row still
//    cover 4 distinct k, so each DMMA is a valid rank-4 update; the sum over
//    the 8 k is unchanged).  For k-contiguous shared tiles (A^T as As[m][k],
//    B as Bs[n][k]) both values come from ONE 16-byte LDS.
//  * row/column pairs.  For m-contiguous tiles (A as As[k][m]) fragment a's
//    lane row is wm0 + 16(a/2) + 2fr + (a%2): fragments 2g and 2g+1 are two
//    adjacent rows, again one 16-byte LDS per k (likewise columns of B^T).
//  * padding that keeps every 8-lane phase of those 16-byte loads on 8
//    distinct 16-byte bank groups: ld = BK + 8 (k-contiguous tiles, 8 mod 16)
//    and ld = BM + 2 / BN + 2 (m/n-contiguous tiles, 2 mod 8).
//
// So a warp tile of FM x FN fragments issues FM + FN 16-byte loads per
// 2 FM FN DMMAs (gemm_f64_kernel: 2 (FM + FN) 8-byte loads), fragments are
// double-buffered across k steps, and the operand tiles stream through a
// STAGES-deep cp.async ring.  K is split across blockIdx.z when the output
// grid cannot fill the SMs; partial planes are summed in a fixed order
// (gemm_reduce_kernel), so results are deterministic run to run.


#include "gemm.cuh"

namespace rq {

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES>
struct TcCfgOld {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int kLdA = TA ? BK + 8 : BM + 2;   // TA: As[m][k]; else As[k][m]
  static constexpr int kLdB = TB ? BN + 2 : BK + 8;   // TB: Bs[k][n]; else Bs[n][k]
  static constexpr int kTileA = TA ? BM * kLdA : BK * kLdA;
  static constexpr int kTileB = TB ? BK * kLdB : BN * kLdB;
  static constexpr size_t kSmem = (size_t)STAGES * (kTileA + kTileB) * sizeof(double);
  static_assert(BM % WM == 0 && BN % WN == 0, "warp grid");
  static_assert(BK % 16 == 0, "k tile: 8 mod 16 padding");
  static_assert(BM % 8 == 0 && BN % 8 == 0, "2 mod 8 padding");
  static_assert(TA || FM % 2 == 0, "m-contiguous A needs row pairs");
  static_assert(!TA || WM % 8 == 0, "fragment rows");
  static_assert(!TB || FN % 2 == 0, "n-contiguous B needs column pairs");
};

// logical row of fragment a held by lane row fr (see the header comment)
template <bool TA>
RQ_DEV int tc_row_old(int wm0, int a, int fr) {
  return TA ? wm0 + 8 * a + fr : wm0 + 16 * (a >> 1) + 2 * fr + (a & 1);
}
// logical column of fragment b, MMA column j
template <bool TB>
RQ_DEV int tc_col_old(int wn0, int b, int j) {
  return TB ? wn0 + 16 * (b >> 1) + 2 * j + (b & 1) : wn0 + 8 * b + j;
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, int VEC,
          int MINB = 1, bool DBUF = true>
__global__ void __launch_bounds__(TcCfgOld<TA, TB, BM, BN, BK, WM, WN, STAGES>::kThreads, MINB)
    tc_gemm_kernel_old(GemmArgs g) {
  using Cfg = TcCfgOld<TA, TB, BM, BN, BK, WM, WN, STAGES>;
  constexpr int NT = Cfg::kThreads, FM = Cfg::FM, FN = Cfg::FN;
  constexpr int LDA = Cfg::kLdA, LDB = Cfg::kLdB;
  if (aborted(g.st)) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::kTileA;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % Cfg::kWarpsM) * WM, wn0 = (warp / Cfg::kWarpsM) * WN;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
  const int64_t kend = imin64(g.K, kbeg + g.kchunk);
  const int ktiles = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  // (outer x inner) tile, inner index contiguous in global memory
  auto copy_tile = [&](double* dst, int lds, const double* src, int64_t ld, int outer, int inner,
                       int64_t o0, int64_t i0, int64_t olim, int64_t ilim) {
    constexpr int V = VEC;
    const int per = inner / V;
#pragma unroll 4
    for (int e = tid; e < outer * per; e += NT) {
      const int o = e / per, i = (e % per) * V;
      const int64_t go = o0 + o, gi = i0 + i;
      const double* p = src + gi + go * ld;
      if (V == 2) {
        const int valid = go < olim ? (gi + 1 < ilim ? 16 : (gi < ilim ? 8 : 0)) : 0;
        cp_async16(dst + o * lds + i, valid ? p : src, valid);
      } else {
        const bool ok = go < olim && gi < ilim;
        cp_async8(dst + o * lds + i, ok ? p : src, ok);
      }
    }
  };
  auto load_tile = [&](int slot, int64_t k0) {
    double* as = As + slot * Cfg::kTileA;
    double* bs = Bs + slot * Cfg::kTileB;
    if (!TA) copy_tile(as, LDA, g.A, g.lda, BK, BM, k0, m0, kend, g.M);   // (k, m)
    else copy_tile(as, LDA, g.A, g.lda, BM, BK, m0, k0, g.M, kend);       // (m, k)
    if (TB) copy_tile(bs, LDB, g.B, g.ldb, BK, BN, k0, n0, kend, g.N);    // (k, n)
    else copy_tile(bs, LDB, g.B, g.ldb, BN, BK, n0, k0, g.N, kend);       // (n, k)
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, kbeg + (int64_t)s * BK);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  // per-lane fragment base offsets inside a stage (k step offsets added later)
  int aoff[TA ? FM : FM / 2], boff[TB ? FN / 2 : FN];
#pragma unroll
  for (int a = 0; a < (TA ? FM : FM / 2); ++a)
    aoff[a] = TA ? (wm0 + 8 * a + fr) * LDA + 2 * fk : (2 * fk) * LDA + wm0 + 16 * a + 2 * fr;
#pragma unroll
  for (int b = 0; b < (TB ? FN / 2 : FN); ++b)
    boff[b] = TB ? (2 * fk) * LDB + wn0 + 16 * b + 2 * fr : (wn0 + 8 * b + fr) * LDB + 2 * fk;

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + STAGES - 1;
      if (pf < ktiles) load_tile(pf % STAGES, kbeg + (int64_t)pf * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::kTileA;
    const double* bs = Bs + (kt % STAGES) * Cfg::kTileB;
    // fragments [buffer][k half][frag]
    double af[2][2][FM], bf[2][2][FN];
    auto ldfrag = [&](int buf, int k8) {
#pragma unroll
      for (int a = 0; a < (TA ? FM : FM / 2); ++a) {
        if (TA) {
          const double2 v = *reinterpret_cast<const double2*>(as + aoff[a] + k8);
          af[buf][0][a] = v.x; af[buf][1][a] = v.y;
        } else {
          const double2 v0 = *reinterpret_cast<const double2*>(as + aoff[a] + k8 * LDA);
          const double2 v1 = *reinterpret_cast<const double2*>(as + aoff[a] + (k8 + 1) * LDA);
          af[buf][0][2 * a] = v0.x; af[buf][0][2 * a + 1] = v0.y;
          af[buf][1][2 * a] = v1.x; af[buf][1][2 * a + 1] = v1.y;
        }
      }
#pragma unroll
      for (int b = 0; b < (TB ? FN / 2 : FN); ++b) {
        if (!TB) {
          const double2 v = *reinterpret_cast<const double2*>(bs + boff[b] + k8);
          bf[buf][0][b] = v.x; bf[buf][1][b] = v.y;
        } else {
          const double2 v0 = *reinterpret_cast<const double2*>(bs + boff[b] + k8 * LDB);
          const double2 v1 = *reinterpret_cast<const double2*>(bs + boff[b] + (k8 + 1) * LDB);
          bf[buf][0][2 * b] = v0.x; bf[buf][0][2 * b + 1] = v0.y;
          bf[buf][1][2 * b] = v1.x; bf[buf][1][2 * b + 1] = v1.y;
        }
      }
    };
    if (DBUF) {
      ldfrag(0, 0);
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        if (ks + 1 < BK / 8) ldfrag((ks + 1) & 1, (ks + 1) * 8);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int b = 0; b < FN; ++b) dmma884(acc[a][b], af[ks & 1][h][a], bf[ks & 1][h][b]);
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        ldfrag(0, ks * 8);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int a = 0; a < FM; ++a)
#pragma unroll
            for (int b = 0; b < FN; ++b) dmma884(acc[a][b], af[0][h][a], bf[0][h][b]);
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: acc[a][b][e] = C[tc_row(a, fr)][tc_col(b, 2 fk + e)]
  const bool split = g.splits > 1;
  double* P = split ? g.partial + (size_t)blockIdx.z * (size_t)(g.M * g.N) : nullptr;
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int64_t r = m0 + tc_row_old<TA>(wm0, a, fr);
    if (r >= g.M) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + tc_col_old<TB>(wn0, b, 2 * fk + e);
        if (c >= g.N) continue;
        if (split) {
          P[r + c * g.M] = acc[a][b][e];
        } else {
          double* cp = g.C + r + c * g.ldc;
          const double old = g.beta == 0.0 ? 0.0 : *cp;
          *cp = gemm_combine(acc[a][b][e], old, g.alpha, g.beta);
        }
      }
    }
  }
}

}  // namespace rq
