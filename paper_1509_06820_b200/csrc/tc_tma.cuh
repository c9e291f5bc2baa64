// TMA-fed variant of tc_gemm_kernel (csrc/tc_gemm.cuh): the operand tiles
// are moved global -> shared by the Tensor Memory Accelerator
// (cp.async.bulk.tensor, one elected thread, mbarrier completion) instead of
// per-thread cp.async, with hardware swizzles in place of padding:
//
//   A (m contiguous) and B^T (n contiguous): boxes of 16 m (n) x 16 k,
//       128-byte swizzle (a 16-byte chunk c of row k lands at c ^ (k & 7));
//   A^T and B (k contiguous): boxes of 8 k x BM (BN) rows, 64-byte swizzle
//       (chunk c of row r lands at c ^ ((r >> 1) & 3)).
//
// The fragment loads are the k-pair / row-pair 16-byte loads of tc_gemm
// (see there), addressed through the same swizzles; every 8-lane phase still
// hits 8 distinct 16-byte bank groups.  Out-of-bounds box elements arrive as
// zeros, so edge tiles need no predication on the load side.  Same
// arithmetic as tc_gemm_kernel (identical DMMA order), same epilogue.
#pragma once

#include <cuda.h>

#include "gemm.cuh"
#include "tc_gemm.cuh"

namespace rq {

RQ_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

RQ_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
RQ_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
RQ_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
RQ_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <bool TA, bool TB, int BM, int BN, int WM, int WN>
struct TmaCfg {
  static constexpr int BK = 16;
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int kBytesA = BM * BK * 8, kBytesB = BN * BK * 8;
  static constexpr int kStage = kBytesA + kBytesB;
  static_assert(BM % 16 == 0 && BN % 16 == 0, "box shapes");
  static_assert(TA || FM % 2 == 0, "m-contiguous A needs row pairs");
  static_assert(!TB || FN % 2 == 0, "n-contiguous B needs column pairs");
  static_assert(kBytesA % 1024 == 0 && kBytesB % 512 == 0, "swizzle atoms");
};

// byte offset of A(m, k) (m, k local to the tile) inside a stage
template <bool TA, int BM>
RQ_DEV int tma_off_a(int m, int k) {
  if (TA) {   // two boxes of 8 k: rows m of 64 bytes, 64-byte swizzle
    const int kk = k & 7;
    return (k >> 3) * (BM * 64) + m * 64 + ((((kk >> 1) ^ (m >> 1)) & 3) << 4) + ((kk & 1) << 3);
  }
  // boxes of 16 m: rows k of 128 bytes, 128-byte swizzle
  return (m >> 4) * 2048 + k * 128 + (((((m & 15) >> 1) ^ k) & 7) << 4) + ((m & 1) << 3);
}
// byte offset of op(B)(k, n): B (k contiguous) like A^T, B^T (n contiguous) like A
template <bool TB, int BN>
RQ_DEV int tma_off_b(int n, int k) {
  return tma_off_a<!TB, BN>(n, k);
}

template <bool TA, bool TB, int BM, int BN, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(TmaCfg<TA, TB, BM, BN, WM, WN>::kThreads, MINB)
    tc_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  GemmArgs g) {
  using Cfg = TmaCfg<TA, TB, BM, BN, WM, WN>;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, BK = Cfg::BK;
  if (aborted(g.st)) return;
  extern __shared__ __align__(16) unsigned char tma_dsm[];
  // swizzle atoms need 1024-byte aligned boxes
  unsigned char* base =
      tma_dsm + ((1024 - (smem_u32(tma_dsm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bars[STAGES];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % Cfg::kWarpsM) * WM, wn0 = (warp / Cfg::kWarpsM) * WN;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
  const int64_t kend = imin64(g.K, kbeg + g.kchunk);
  const int ktiles = kbeg < kend ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int s, int64_t k0) {   // thread 0 only
    unsigned char* st = base + s * Cfg::kStage;
    mbar_expect_tx(&bars[s], Cfg::kStage);
    if (TA) {
#pragma unroll
      for (int b = 0; b < 2; ++b)
        tma_load_2d(st + b * (BM * 64), &tmA, (int)(k0 + 8 * b), (int)m0, &bars[s]);
    } else {
#pragma unroll
      for (int b = 0; b < BM / 16; ++b)
        tma_load_2d(st + b * 2048, &tmA, (int)(m0 + 16 * b), (int)k0, &bars[s]);
    }
    if (!TB) {
#pragma unroll
      for (int b = 0; b < 2; ++b)
        tma_load_2d(st + Cfg::kBytesA + b * (BN * 64), &tmB, (int)(k0 + 8 * b), (int)n0, &bars[s]);
    } else {
#pragma unroll
      for (int b = 0; b < BN / 16; ++b)
        tma_load_2d(st + Cfg::kBytesA + b * 2048, &tmB, (int)(n0 + 16 * b), (int)k0, &bars[s]);
    }
  };

  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  if (tid == 0)
    for (int s = 0; s < STAGES - 1 && s < ktiles; ++s) issue(s, kbeg + (int64_t)s * BK);
  const int fr = lane >> 2, fk = lane & 3;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&bars[s], (unsigned)((kt / STAGES) & 1));
    __syncthreads();   // every warp is done with stage (kt - 1) % STAGES
    if (tid == 0 && kt + STAGES - 1 < ktiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue((kt + STAGES - 1) % STAGES, kbeg + (int64_t)(kt + STAGES - 1) * BK);
    }
    const unsigned char* sa = base + s * Cfg::kStage;
    const unsigned char* sb = sa + Cfg::kBytesA;
#pragma unroll
    for (int ks = 0; ks < BK / 8; ++ks) {
      const int k8 = ks * 8;
      double af[2][FM], bf[2][FN];
#pragma unroll
      for (int a = 0; a < (TA ? FM : FM / 2); ++a) {
        if (TA) {
          const double2 v = *reinterpret_cast<const double2*>(
              sa + tma_off_a<true, BM>(wm0 + 8 * a + fr, k8 + 2 * fk));
          af[0][a] = v.x; af[1][a] = v.y;
        } else {
          const int m = wm0 + 16 * a + 2 * fr;
          const double2 v0 = *reinterpret_cast<const double2*>(sa + tma_off_a<false, BM>(m, k8 + 2 * fk));
          const double2 v1 =
              *reinterpret_cast<const double2*>(sa + tma_off_a<false, BM>(m, k8 + 2 * fk + 1));
          af[0][2 * a] = v0.x; af[0][2 * a + 1] = v0.y;
          af[1][2 * a] = v1.x; af[1][2 * a + 1] = v1.y;
        }
      }
#pragma unroll
      for (int b = 0; b < (TB ? FN / 2 : FN); ++b) {
        if (!TB) {
          const double2 v = *reinterpret_cast<const double2*>(
              sb + tma_off_b<false, BN>(wn0 + 8 * b + fr, k8 + 2 * fk));
          bf[0][b] = v.x; bf[1][b] = v.y;
        } else {
          const int n = wn0 + 16 * b + 2 * fr;
          const double2 v0 = *reinterpret_cast<const double2*>(sb + tma_off_b<true, BN>(n, k8 + 2 * fk));
          const double2 v1 =
              *reinterpret_cast<const double2*>(sb + tma_off_b<true, BN>(n, k8 + 2 * fk + 1));
          bf[0][2 * b] = v0.x; bf[0][2 * b + 1] = v0.y;
          bf[1][2 * b] = v1.x; bf[1][2 * b + 1] = v1.y;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int a = 0; a < FM; ++a)
#pragma unroll
          for (int b = 0; b < FN; ++b) dmma884(acc[a][b], af[h][a], bf[h][b]);
    }
  }

  // epilogue (tc_gemm_kernel's): acc[a][b][e] = C[tc_row(a, fr)][tc_col(b, 2 fk + e)]
  const bool split = g.splits > 1;
  if (!split && g.beta != 0.0) {
#pragma unroll
    for (int a = 0; a < FM; ++a) {
      const int64_t r = m0 + tc_row<TA>(wm0, a, fr);
      if (r >= g.M) continue;
      double old[FN][2];
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + tc_col<TB>(wn0, b, 2 * fk + e);
          old[b][e] = c < g.N ? __ldcg(g.C + r + c * g.ldc) : 0.0;
        }
#pragma unroll
      for (int b = 0; b < FN; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = n0 + tc_col<TB>(wn0, b, 2 * fk + e);
          if (c < g.N) g.C[r + c * g.ldc] = gemm_combine(acc[a][b][e], old[b][e], g.alpha, g.beta);
        }
    }
    return;
  }
  double* P = split ? g.partial + (size_t)blockIdx.z * (size_t)(g.M * g.N) : nullptr;
#pragma unroll
  for (int a = 0; a < FM; ++a) {
    const int64_t r = m0 + tc_row<TA>(wm0, a, fr);
    if (r >= g.M) continue;
#pragma unroll
    for (int b = 0; b < FN; ++b) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = n0 + tc_col<TB>(wn0, b, 2 * fk + e);
        if (c >= g.N) continue;
        if (split) P[r + c * g.M] = acc[a][b][e];
        else g.C[r + c * g.ldc] = gemm_combine(acc[a][b][e], 0.0, g.alpha, 0.0);
      }
    }
  }
}

}  // namespace rq
