// Small dense triangular helpers on the FP64 tensor pipe, shared by the
// fast panel (panel_fast.cu) and the sample update (small.cu).
#pragma once

#include "gemm.cuh"

namespace rq {

// one 8x8 output tile: acc += A(8 x K) B(K x 8), A/B row-major (stride ld)
// at their tile origins, K a multiple of 4
RQ_DEV void tile_mm(const double* A, const double* B, int K, int ld, double (&acc)[2]) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  for (int k4 = 0; k4 < K; k4 += 4) dmma884(acc, A[fr * ld + k4 + fk], B[(k4 + fk) * ld + fr]);
}
RQ_DEV void tile_store(double* C, int ld, const double (&acc)[2], double scale) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  C[fr * ld + 2 * fk] = scale * acc[0];
  C[fr * ld + 2 * fk + 1] = scale * acc[1];
}

// X = U^{-1} for an upper triangular n8 x n8 U, n8 in {8, 16, 32, 64} (the
// levels join pairs of equal blocks; row-major, stride ld; the
// padding beyond n is the identity; dinv[j] = 1 / U[j][j] for j < n8).
// Recursive block inverse: warp w inverts diagonal block w (8 x 8, one
// column per lane, in registers), then levels s = 8, 16, 32 join pairs of
// s-blocks with  X12 = -X11 (U12 X22)  on the FP64 tensor pipe.
template <int NT>
RQ_DEV void upper_inverse(const double* U, const double* dinv, double* X, double* Tmp, int n8,
                          int ld) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < n8 * n8; e += NT) {
    const int i = e / n8, l = e - i * n8;
    if ((i >> 3) != (l >> 3)) X[i * ld + l] = 0.0;
  }
  if (warp < n8 / 8) {
    const int b0 = 8 * warp, c = lane & 7;
    double x[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) x[r] = (r == c) ? 1.0 : 0.0;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      x[j] *= dinv[b0 + j];
#pragma unroll
      for (int i = 0; i < j; ++i) x[i] = __fma_rn(-U[(b0 + i) * ld + b0 + j], x[j], x[i]);
    }
    if (lane < 8)
#pragma unroll
      for (int r = 0; r < 8; ++r) X[(b0 + r) * ld + b0 + c] = x[r];
  }
  __syncthreads();
  for (int sz = 8; sz < n8; sz *= 2) {
    const int tpb = sz / 8, per = tpb * tpb, ntile = (n8 / (2 * sz)) * per;
    // T = U12 X22 (into Tmp at the X12 position)
    for (int t = warp; t < ntile; t += NT / 32) {
      const int p = t / per, ti = (t % per) / tpb, tj = t % tpb;
      const int r0 = 2 * p * sz + 8 * ti, d0 = 2 * p * sz + sz, c0 = d0 + 8 * tj;
      double acc[2] = {0.0, 0.0};
      tile_mm(U + r0 * ld + d0, X + d0 * ld + c0, 8 * (tj + 1), ld, acc);   // X22 upper
      tile_store(Tmp + r0 * ld + c0, ld, acc, 1.0);
    }
    __syncthreads();
    // X12 = -X11 T
    for (int t = warp; t < ntile; t += NT / 32) {
      const int p = t / per, ti = (t % per) / tpb, tj = t % tpb;
      const int a0 = 2 * p * sz, r0 = a0 + 8 * ti, c0 = a0 + sz + 8 * tj;
      double acc[2] = {0.0, 0.0};
      tile_mm(X + r0 * ld + r0, Tmp + r0 * ld + c0, sz - 8 * ti, ld, acc);  // X11 upper
      tile_store(X + r0 * ld + c0, ld, acc, -1.0);
    }
    __syncthreads();
  }
}


}  // namespace rq
