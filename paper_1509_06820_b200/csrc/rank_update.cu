// K2: persistent rank-b trailing update  C -= Y X  (K = b <= 64), the second
// half of _block_stages (randomized.py:174-178: R12 = C[:b] - Y[:b] X and
// C[b:] -= Y[b:] X in one pass over all rows).
//
// The generic DMMA GEMM stalls on its epilogue C reads here (ncu: long
// scoreboard, tensor pipe 33% active): with K = 64 the main loop is only 16
// DMMA k-steps, so nothing hides the C round trip.  This kernel runs one CTA
// per SM over a contiguous range of 64x64 output tiles (consecutive tiles
// share their X column block) and double-buffers Y, X and the C tile itself
// with cp.async: while the DMMAs of tile t run, tile t+1's operands are in
// flight.  The epilogue reads C from shared memory and writes C - acc with a
// separate subtraction (numpy's `C - Y @ X` rounding).
#include "gemm.cuh"
#include "runtime.hpp"

namespace rq {

namespace {

constexpr int kTM = 64, kTN = 64, kKMax = 64;
constexpr int kRuThreads = 256;            // 8 warps: 2 (M) x 4 (N), warp tile 32 x 16
constexpr int kLdA = kTM + 4;              // As[k][m]
constexpr int kLdB = kKMax + 4;            // Bs[n][k]
constexpr int kLdC = kTM + 4;              // Cs[n][m]
constexpr int kStageA = kKMax * kLdA, kStageB = kTN * kLdB, kStageC = kTN * kLdC;
constexpr size_t kRuSmem = (size_t)2 * (kStageA + kStageB + kStageC) * sizeof(double);

struct RuArgs {
  int64_t M, N;
  int K;
  const double* Y; int64_t ldy;
  const double* X; int64_t ldx;
  double* C; int64_t ldc;
  const Status* st;
};

__global__ void __launch_bounds__(kRuThreads, 1) rank_update_kernel(RuArgs a) {
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = As + 2 * kStageA;
  double* Cs = Bs + 2 * kStageB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 16;
  const int fr = lane >> 2, fk = lane & 3;
  const int K = a.K;
  const int64_t tm = (a.M + kTM - 1) / kTM, tn = (a.N + kTN - 1) / kTN;
  const int64_t ntiles = tm * tn;
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_hi = ntiles * (blockIdx.x + 1) / gridDim.x;

  // issue the async loads of tile t into buffer b (X only when its column
  // block differs from the one already in that buffer's slot)
  auto load_tile = [&](int64_t t, int b) {
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    double* as = As + b * kStageA;
    double* bs = Bs + b * kStageB;
    double* cs = Cs + b * kStageC;
    // Y[m0:m0+64, 0:K] -> As[k][m]
    for (int e = tid; e < kTM * K; e += kRuThreads) {
      const int i = e % kTM, k = e / kTM;
      const int64_t gi = m0 + i;
      const bool ok = gi < a.M;
      cp_async8(as + k * kLdA + i, ok ? a.Y + gi + k * a.ldy : a.Y, ok);
    }
    // X[0:K, n0:n0+64] -> Bs[n][k]
    for (int e = tid; e < kTN * K; e += kRuThreads) {
      const int k = e % K, j = e / K;
      const int64_t gj = n0 + j;
      const bool ok = gj < a.N;
      cp_async8(bs + j * kLdB + k, ok ? a.X + k + gj * a.ldx : a.X, ok);
    }
    // C[m0:m0+64, n0:n0+64] -> Cs[n][m]
    for (int e = tid; e < kTM * kTN; e += kRuThreads) {
      const int i = e % kTM, j = e / kTM;
      const int64_t gi = m0 + i, gj = n0 + j;
      const bool ok = gi < a.M && gj < a.N;
      cp_async8(cs + j * kLdC + i, ok ? a.C + gi + gj * a.ldc : a.C, ok);
    }
    cp_async_commit();
  };

  if (t_lo < t_hi) load_tile(t_lo, 0);
  int buf = 0;
  for (int64_t t = t_lo; t < t_hi; ++t, buf ^= 1) {
    if (t + 1 < t_hi) {
      load_tile(t + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + buf * kStageA;
    const double* bs = Bs + buf * kStageB;
    const double* cs = Cs + buf * kStageC;
    double acc[4][2][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    for (int k4 = 0; k4 < K; k4 += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int x = 0; x < 4; ++x) af[x] = as[(k4 + fk) * kLdA + wm0 + x * 8 + fr];
#pragma unroll
      for (int y = 0; y < 2; ++y) bf[y] = bs[(wn0 + y * 8 + fr) * kLdB + k4 + fk];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) dmma884(acc[x][y], af[x], bf[y]);
    }
    // epilogue: C - acc (C from shared memory)
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int i = wm0 + x * 8 + fr;
      const int64_t gi = m0 + i;
      if (gi >= a.M) continue;
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = wn0 + y * 8 + 2 * fk + e;
          const int64_t gj = n0 + j;
          if (gj < a.N) a.C[gi + gj * a.ldc] = __dsub_rn(cs[j * kLdC + i], acc[x][y][e]);
        }
    }
    __syncthreads();  // buffer `buf` is reloaded by the next iteration's prefetch
  }
}

}  // namespace

bool rank_update(Handle& h, int64_t M, int64_t N, int64_t K, const double* Y, int64_t ldy,
                 const double* X, int64_t ldx, double* C, int64_t ldc, cudaStream_t s,
                 const Status* st, int cat) {
  if (K < 4 || K > kKMax || (K % 4) != 0 || M <= 0 || N <= 0) return false;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA(cudaFuncSetAttribute(rank_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kRuSmem));
    attr = true;
  }
  RuArgs a{M, N, (int)K, Y, ldy, X, ldx, C, ldc, st};
  const int64_t ntiles = ((M + kTM - 1) / kTM) * ((N + kTN - 1) / kTN);
  const int grid = (int)std::min<int64_t>(h.num_sms, ntiles);
  ProfScope prof(h, cat, 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + 2.0 * M * N), s);
  rank_update_kernel<<<grid, kRuThreads, kRuSmem, s>>>(a);
  RQ_CHECK_LAUNCH();
  count_launch();
  return true;
}

}  // namespace rq
