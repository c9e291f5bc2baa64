// K7: the rest of a speculative RQRCP block after a committed fast panel
// (randomized.py:158-180 _block_stages up to R12, and randomized.py:107-135
// sample_update), fused per 64-column tile of the trailing matrix:
//
//   X_c   = A1^T C_top,c + A2^T H_c          (= T^T (Y^T C)_c, A1 = Y1 T, A2 = M T)
//   R12_c = C_top,c - Y_top X_c              (written in place, rows i0..i0+b)
//   B_c   = [S12_c - Msu R12_c ; S22_c]      (Msu = S11 R11^{-1}, from the panel)
//
// Every column tile is independent, so one launch replaces the two G-assembly
// GEMMs, X = T^T G, the R12 update, the sample update and the panel's zero
// fill that sat on the per-block critical path (~35 us of latency-bound
// launches).  Each product is b x 64 x K on the FP64 tensor pipe, operands
// staged in shared memory; the trailing update (C[b:] -= Y[b:] X) then runs
// on the side-stream-overlapped path with X from here.
#include "gemm.cuh"
#include "runtime.hpp"

namespace rq {

namespace {

constexpr int kFinT = 256;   // 8 warps: 2 (m) x 4 (n), warp tile 32 x 16
// columns per CTA: 64, or 32 when 64-wide tiles would leave SMs idle (the
// three products are DMMA-throughput bound per SM: ~2 MFLOP per 64-wide tile)
constexpr int kFinLd = 68;   // k-major A operands: [k][m], row stride (doubles)

// acc(64 x 64 tile, this warp's 32 x 16) += A B: A-fragment (m, k) at
// Ak[k * kFinLd + m] (k-major), B-fragment (k, n) at Bn[n * ldb + k] (n-major,
// ldb = 8 mod 16 words apart per n: conflict-free 64-bit fragment loads);
// fragments double-buffered in registers
template <int K, int YN>
RQ_DEV void tile_prod(const double* Ak, const double* Bn, int ldb, double (&acc)[4][YN][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 8 * YN;
  const int fr = lane >> 2, fk = lane & 3;
  double af[2][4], bf[2][YN];
  auto load = [&](int k4, int p) {
#pragma unroll
    for (int x = 0; x < 4; ++x) af[p][x] = Ak[(k4 + fk) * kFinLd + wm0 + x * 8 + fr];
#pragma unroll
    for (int y = 0; y < YN; ++y) bf[p][y] = Bn[(wn0 + y * 8 + fr) * ldb + k4 + fk];
  };
  load(0, 0);
#pragma unroll
  for (int k4 = 0; k4 < K; k4 += 4) {
    const int p = (k4 >> 2) & 1;
    if (k4 + 4 < K) load(k4 + 4, p ^ 1);
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < YN; ++y) dmma884(acc[x][y], af[p][x], bf[p][y]);
  }
}

template <int YN>
RQ_DEV void zero_acc(double (&acc)[4][YN][2]) {
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < YN; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
}

// column segment of `len` doubles (len even) global -> shared, 16-byte copies
// when both ends are 16-byte aligned, else 8-byte; `ok` false zero-fills
RQ_DEV void stage_col(double* dst, const double* src, int len, bool ok, int lane, int nl) {
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (al) {
    for (int i = 2 * lane; i < len; i += 2 * nl) cp_async16(dst + i, ok ? src + i : src, ok ? 16 : 0);
  } else {
    for (int i = lane; i < len; i += nl) cp_async8(dst + i, ok ? src + i : src, ok);
  }
}

template <int B, int NW>
__global__ void __launch_bounds__(kFinT, 1) block_finish_kernel(FinishArgs a) {
  constexpr int kFinN = NW, YN = NW / 32;
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.pre != nullptr)
    a.pre->abort = *((volatile const int*)&a.st->abort);   // predicate of the trailing update
  if (aborted(a.st)) return;
  constexpr int LB = 2 * B + 4;      // n-major row stride of the B operands ([C_top; H] / [R12; X])
  constexpr int LS = B + 4;          // S12 as [n][m]
  extern __shared__ __align__(16) double fsm[];
  double* AK = fsm;                  // [2B][kFinLd]  [A1; A2] (k-major)
  double* BN = AK + 2 * B * kFinLd;  // [64][LB]      [C_top; H] per column; later [R12; X]
  double* YT = BN + kFinN * LB;      // [B][kFinLd]   YT[k][m] = Y_top(m, k)
  double* MS = YT + B * kFinLd;      // [B][kFinLd]   MS[k][m] = Msu(m, k)
  double* SS = AK;                   // [64][LS]      S12 per column, after phase 1
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 8 * YN;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t c0 = (int64_t)blockIdx.x * kFinN;
  const int nc = (int)imin64(kFinN, a.nt2 - c0);

  // every operand of the three products in flight at once
  for (int e = 2 * tid; e < 2 * B * B; e += 2 * kFinT)   // A12 is row-major [k][m]
    cp_async16(&AK[(e / B) * kFinLd + e % B], a.A12 + e, 16);
  for (int k = warp; k < B; k += kFinT / 32) {           // one column of Y_top / Msu per warp
    stage_col(&YT[k * kFinLd], a.Ytop + (int64_t)k * a.ldy, B, true, lane, 32);
    stage_col(&MS[k * kFinLd], a.Msu + (int64_t)k * B, B, true, lane, 32);
  }
  for (int n = warp; n < kFinN; n += kFinT / 32) {       // per trailing column: C_top, H
    const bool ok = n < nc;
    const int64_t cn = ok ? c0 + n : 0;
    stage_col(&BN[n * LB], a.Ctop + cn * a.ldw, B, ok, lane, 32);
    stage_col(&BN[n * LB + B], a.H + cn * B, B, ok, lane, 32);
  }
  cp_async_commit();
  if (B < 64)   // m past B: zero A operands so the idle accumulators stay finite
    for (int e = tid; e < 2 * B * (64 - B); e += kFinT) {
      const int k = e / (64 - B), m = B + e % (64 - B);
      AK[k * kFinLd + m] = 0.0;
      if (k < B) YT[k * kFinLd + m] = MS[k * kFinLd + m] = 0.0;
    }
  {   // zero fill of the panel rows below the diagonal: (column, 1024-row chunk) items
    const int rows = (int)(a.mm - B), chunks = (rows + 1023) >> 10;
    for (int it = blockIdx.x; it < B * chunks; it += gridDim.x) {
      const int c = it / chunks, r0 = (it - c * chunks) << 10, r1 = min(rows, r0 + 1024);
      double* col = a.Pz + (int64_t)c * a.ldw;
      for (int r = r0 + tid; r < r1; r += kFinT) col[r] = 0.0;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  double acc[4][YN][2];
  // ---- X = [A1; A2]^T [C_top; H]
  zero_acc(acc);
  tile_prod<2 * B, YN>(AK, BN, LB, acc);
  __syncthreads();   // AK and the H part of BN are free
  for (int n = warp; n < kFinN; n += kFinT / 32) {       // S12, lands during phase 2
    const bool ok = n < nc;
    stage_col(&SS[n * LS], a.S + (ok ? c0 + n : 0) * a.lds, B, ok, lane, 32);
  }
  cp_async_commit();
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < YN; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = wm0 + x * 8 + fr, n = wn0 + y * 8 + 2 * fk + e;
        if (m < B) {
          BN[n * LB + B + m] = acc[x][y][e];
          if (n < nc) a.X[m + (c0 + n) * B] = acc[x][y][e];
        }
      }
  __syncthreads();
  // ---- R12 = C_top - Y_top X  (C_top part of BN overwritten in place by its owner)
  zero_acc(acc);
  tile_prod<B, YN>(YT, BN + B, LB, acc);
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < YN; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = wm0 + x * 8 + fr, n = wn0 + y * 8 + 2 * fk + e;
        if (m < B) {
          const double r = __dsub_rn(BN[n * LB + m], acc[x][y][e]);
          BN[n * LB + m] = r;   // zero past nc (C_top and X are zero there)
          if (n < nc) a.Ctop[m + (c0 + n) * a.ldw] = r;
        }
      }
  cp_async_wait<0>();
  __syncthreads();
  // ---- B_new = [S12 - Msu R12; S22]
  zero_acc(acc);
  tile_prod<B, YN>(MS, BN, LB, acc);
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < YN; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = wm0 + x * 8 + fr, n = wn0 + y * 8 + 2 * fk + e;
        if (m < B && n < nc)
          a.Bn[m + (c0 + n) * a.ldb] = __dsub_rn(SS[n * LS + m], acc[x][y][e]);
      }
  const int r22 = a.ell - B;
  for (int e = tid; e < r22 * nc; e += kFinT) {
    const int n = e / r22, r = B + e % r22;
    a.Bn[r + (c0 + n) * a.ldb] = a.S[r + (c0 + n) * a.lds];
  }
  if (a.done_ctr != nullptr) {
    // randomized.py:117 raised: the block stays committed (R12 above, the
    // trailing update on its snapshot predicate), the sample update is void
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
        *a.done_ctr = 0;
        if (*((volatile const int*)&a.st->degenerate) != 0) {
          a.st->abort_i0 = a.i0;
          __threadfence();
          a.st->abort = kAbortDegenerate;
        }
      }
    }
  }
}

template <int B, int NW>
void launch_finish(const FinishArgs& f, cudaStream_t s) {
  constexpr size_t smem = ((size_t)4 * B * kFinLd + (size_t)NW * (2 * B + 4)) * sizeof(double);
  kernel_attr((const void*)block_finish_kernel<B, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)smem);
  const int grid = (int)((f.nt2 + NW - 1) / NW);
  block_finish_kernel<B, NW><<<grid, kFinT, smem, s>>>(f);
}

}  // namespace

bool block_finish(Handle& h, const FinishArgs& f, cudaStream_t s) {
  if ((f.b != 32 && f.b != 64) || f.nt2 <= 0 || f.ell < f.b) return false;
  ProfScope prof(h, kProfSmallGemm, 2.0 * f.b * f.nt2 * (2.0 * f.b + f.b + f.b),
                 8.0 * (4.0 * f.b * f.nt2 + (double)f.ell * f.nt2), s);
  // 32-wide tiles while 64-wide ones would not fill the SMs
  const bool narrow = h.finish_narrow && (f.nt2 + 63) / 64 < h.num_sms;
  if (f.b == 64) {
    if (narrow) launch_finish<64, 32>(f, s);
    else launch_finish<64, 64>(f, s);
  } else {
    if (narrow) launch_finish<32, 32>(f, s);
    else launch_finish<32, 64>(f, s);
  }
  RQ_CHECK_LAUNCH();
  count_launch();
  return true;
}

}  // namespace rq
