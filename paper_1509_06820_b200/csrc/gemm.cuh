// FP64 tensor-core GEMM for sm_100a: C = alpha * op(A) op(B) + beta * C.
//
// sm_100a has no FP64 tcgen05 kind (CUDA 12.9 tcgen05_mma.h lists only
// f16/tf32/f8f6f4/i8/mxf*), so the FP64 tensor path is the warp-level
// `mma.sync.m8n8k4.f64` (SASS DMMA.8x8x4).  Operand tiles are staged
// global->shared with cp.async (LDGSTS, zero-filled at the edges) in a
// multi-stage ring; the shared tiles are k-major with a +4 double pad so the
// DMMA fragment loads (8 rows x 4 k per warp) are bank-conflict free.
//
// Used for every level-3 call site of the hot path:
//   sketch      B = Omega A                  (randomized.py:76, truncated.py:59)
//   stage 1     G = Y^T C, X = T^T G          (randomized.py:172; truncated.py:144-149)
//   stage 2/3   C -= Y X  (R12 rows + trailing)  (randomized.py:174-178)
//   TRQRCP      panel / R-row materialisation  (truncated.py:121, 152-155)
//   TUXV        A V, block reflections, Q formation (truncated.py:230; qrcp.py:53-60, 222-252)
// K is split across blockIdx.z when the output tile grid is too small to fill
// 148 SMs; partial tiles go to a workspace and are summed in fixed split order
// by gemm_reduce_kernel, so results are deterministic run to run.
#pragma once

#include "common.cuh"

namespace rq {

struct GemmArgs {
  int64_t M, N, K;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  double* C; int64_t ldc;
  double alpha, beta;
  int splits;          // number of K chunks (blockIdx.z)
  int64_t kchunk;      // K per chunk (multiple of BK)
  double* partial;     // splits > 1: [splits][M x N], ld = M
  const Status* st;    // abort predicate, may be null
};

RQ_DEV void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
// 16-byte copy of up to two doubles; bytes beyond `valid` (0, 8, 16) are zero-filled
RQ_DEV void cp_async16(void* smem, const void* gmem, int valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid));
}
RQ_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RQ_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

RQ_DEV void dmma884(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// epilogue combine, written to match numpy's separately rounded
// `C - Y @ X` / `alpha * (A @ B)` forms (no FMA contraction)
RQ_DEV double gemm_combine(double acc, double c, double alpha, double beta) {
  if (beta == 0.0) return alpha == 1.0 ? acc : __dmul_rn(alpha, acc);
  if (alpha == -1.0 && beta == 1.0) return __dsub_rn(c, acc);
  if (alpha == 1.0 && beta == 1.0) return __dadd_rn(c, acc);
  return __dadd_rn(__dmul_rn(alpha, acc), __dmul_rn(beta, c));
}

// Shared tiles follow the operand's contiguous global direction so every
// copy is contiguous on both sides (16-byte cp.async when aligned, no write
// bank conflicts):
//   A: !TA -> As[k][m] (ld BM+4)     TA -> As[m][k] (ld BK+4)
//   B:  TB -> Bs[k][n] (ld BN+4)    !TB -> Bs[n][k] (ld BK+4)
// Each padded leading dimension is 4 (mod 16) doubles, so the DMMA fragment
// loads (8 rows x 4 k per warp) hit distinct banks within each half-warp.
template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  static constexpr int kLdA = TA ? BK + 4 : BM + 4;
  static constexpr int kLdB = TB ? BN + 4 : BK + 4;
  static constexpr int kTileA = TA ? BM * kLdA : BK * kLdA;
  static constexpr int kTileB = TB ? BK * kLdB : BN * kLdB;
  static constexpr size_t kSmem = (size_t)STAGES * (kTileA + kTileB) * sizeof(double);
  static_assert(BM % 16 == 0 && BN % 16 == 0 && BK % 16 == 0, "pad trick needs multiples of 16");
  static_assert(WM % 8 == 0 && WN % 8 == 0, "fragment shape");
};

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, int VEC>
__global__ void __launch_bounds__(GemmCfg<TA, TB, BM, BN, BK, WM, WN, STAGES>::kThreads)
    gemm_f64_kernel(GemmArgs g) {
  using Cfg = GemmCfg<TA, TB, BM, BN, BK, WM, WN, STAGES>;
  constexpr int NT = Cfg::kThreads;
  constexpr int FM = WM / 8, FN = WN / 8;
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

  // copy an (outer x inner) tile whose inner index is contiguous in global
  // memory (element (o, i) at src + i + o * ld) into dst[o * lds + i]
  auto copy_tile = [&](double* dst, int lds, const double* src, int64_t ld, int outer, int inner,
                       int64_t o0, int64_t i0, int64_t olim, int64_t ilim) {
    constexpr int V = VEC;
    const int per = inner / V;
#pragma unroll
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
    if (!TA) copy_tile(as, Cfg::kLdA, g.A, g.lda, BK, BM, k0, m0, kend, g.M);   // (k, m)
    else copy_tile(as, Cfg::kLdA, g.A, g.lda, BM, BK, m0, k0, g.M, kend);       // (m, k)
    if (TB) copy_tile(bs, Cfg::kLdB, g.B, g.ldb, BK, BN, k0, n0, kend, g.N);    // (k, n)
    else copy_tile(bs, Cfg::kLdB, g.B, g.ldb, BN, BK, n0, k0, g.N, kend);       // (n, k)
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
    // fragments double-buffered in registers: step ks+1's loads are issued
    // before step ks's DMMAs (reusing one fragment set made every load wait
    // for the DMMA that last read its register -- ncu source view)
    double af[2][FM], bf[2][FN];
    auto ldfrag = [&](int buf, int k4) {
#pragma unroll
      for (int a = 0; a < FM; ++a) {
        const int m = wm0 + a * 8 + fr, k = k4 + fk;
        af[buf][a] = TA ? as[m * Cfg::kLdA + k] : as[k * Cfg::kLdA + m];
      }
#pragma unroll
      for (int b = 0; b < FN; ++b) {
        const int n = wn0 + b * 8 + fr, k = k4 + fk;
        bf[buf][b] = TB ? bs[k * Cfg::kLdB + n] : bs[n * Cfg::kLdB + k];
      }
    };
    ldfrag(0, 0);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      if (ks + 1 < BK / 4) ldfrag((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int a = 0; a < FM; ++a)
#pragma unroll
        for (int b = 0; b < FN; ++b) dmma884(acc[a][b], af[ks & 1][a], bf[ks & 1][b]);
    }
  }
  cp_async_wait<0>();

  // epilogue: lane holds C[fr][2*fk + e] of each 8x8 fragment
  const bool split = g.splits > 1;
  double* P = split ? g.partial + (size_t)blockIdx.z * (size_t)(g.M * g.N) : nullptr;
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int64_t r = m0 + wm0 + a * 8 + fr;
    if (r >= g.M) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + wn0 + b * 8 + 2 * fk + e;
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

// Deterministic split-K reduction: sum partial[0..splits) in order.
__global__ void gemm_reduce_kernel(GemmArgs g);

}  // namespace rq
