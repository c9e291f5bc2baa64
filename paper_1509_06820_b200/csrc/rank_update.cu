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
  int vec16;
  Status* snap;   // optional: copy of st->abort taken at kernel entry (block 0)
  // optional (K-specialised kernel): C is read from Cs (ld ldcs) and written
  // to C, and rows [M, M + extra_rows) of Cs are copied through unchanged
  const double* Cs; int64_t ldcs; int extra_rows;
};

RQ_DEV void snapshot_abort(const RuArgs& a) {
  if (a.snap != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    a.snap->abort = a.st != nullptr ? *((volatile const int*)&a.st->abort) : 0;
}

__global__ void __launch_bounds__(kRuThreads, 1) rank_update_kernel(RuArgs a) {
  snapshot_abort(a);
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

  // async loads of tile t: Y and C into buffer b; X into X slot xs only when
  // the tile starts a new column block (consecutive tiles share X)
  const bool vec = a.vec16;
  auto copy2d = [&](double* dst, int lds, const double* src, int64_t ld, int outer, int inner,
                    int64_t o0, int64_t i0, int64_t olim, int64_t ilim) {
    if (vec) {
      const int per = inner / 2;
      for (int e = tid; e < outer * per; e += kRuThreads) {
        const int o = e / per, i = (e % per) * 2;
        const int64_t go = o0 + o, gi = i0 + i;
        const int valid = go < olim ? (gi + 1 < ilim ? 16 : (gi < ilim ? 8 : 0)) : 0;
        cp_async16(dst + o * lds + i, valid ? src + gi + go * ld : src, valid);
      }
    } else {
      for (int e = tid; e < outer * inner; e += kRuThreads) {
        const int o = e / inner, i = e % inner;
        const int64_t go = o0 + o, gi = i0 + i;
        const bool ok = go < olim && gi < ilim;
        cp_async8(dst + o * lds + i, ok ? src + gi + go * ld : src, ok);
      }
    }
  };
  auto load_tile = [&](int64_t t, int b, int xs, bool load_x) {
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    copy2d(As + b * kStageA, kLdA, a.Y, a.ldy, K, kTM, 0, m0, K, a.M);          // As[k][m]
    if (load_x) copy2d(Bs + xs * kStageB, kLdB, a.X, a.ldx, kTN, K, n0, 0, a.N, K);  // Bs[n][k]
    copy2d(Cs + b * kStageC, kLdC, a.C, a.ldc, kTN, kTM, n0, m0, a.N, a.M);     // Cs[n][m]
    cp_async_commit();
  };

  int xs = 0;
  if (t_lo < t_hi) load_tile(t_lo, 0, 0, true);
  int buf = 0;
  for (int64_t t = t_lo; t < t_hi; ++t, buf ^= 1) {
    int xs_next = xs;
    if (t + 1 < t_hi) {
      const bool newx = (t + 1) / tm != t / tm;
      if (newx) xs_next = xs ^ 1;
      load_tile(t + 1, buf ^ 1, xs_next, newx);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + buf * kStageA;
    const double* bs = Bs + xs * kStageB;
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
    __syncthreads();  // buffers `buf` / X slot reloaded by the next prefetch
    xs = xs_next;
  }
}

// Specialisation for the block widths in use (K = 32, 64) with 16-byte
// aligned operands: the k-loop unrolls to immediate shared-memory offsets and
// every thread's cp.async pattern within a tile is fixed, so a tile's copies
// are a base pointer plus constant strides (the generic kernel above spends
// ~45% of its issue slots on per-element address arithmetic -- ncu source
// counters, profiles/).  Edge tiles take the checked path.
template <int K>
__global__ void __launch_bounds__(kRuThreads, 1) rank_update_k_kernel(RuArgs a) {
  snapshot_abort(a);
  if (aborted(a.st)) return;
  constexpr int LDB = K + 4;
  constexpr int SA = K * kLdA, SB = kTN * LDB, SC = kTN * kLdC;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = As + 2 * SA;
  double* Cs = Bs + 2 * SB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 16;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t M = a.M, N = a.N;
  const int64_t tm = (M + kTM - 1) / kTM, tn = (N + kTN - 1) / kTN;
  const int64_t ntiles = tm * tn;
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int64_t ldy = a.ldy, ldx = a.ldx, ldc = a.ldc;
  const double* Csrc = a.Cs != nullptr ? a.Cs : a.C;
  const int64_t ldcs = a.Cs != nullptr ? a.ldcs : a.ldc;
  // fixed per-thread copy pattern (16 B per cp.async)
  //   Y tile As[k][m]: k = (tid >> 5) + 8 q, m = 2 (tid & 31)        q < K / 8
  //   C tile Cs[n][m]: n = (tid >> 5) + 8 q, m = 2 (tid & 31)        q < 8
  //   X tile Bs[n][k]: per = K / 2 pairs per column
  constexpr int XPER = K / 2, XROWS = kRuThreads / XPER;   // columns per pass
  const int ym = 2 * (tid & 31), yk = tid >> 5;
  const int xk = 2 * (tid % XPER), xn = tid / XPER;
  auto load_full = [&](int64_t t, int b, int xs, bool load_x) {
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    {
      const double* g = a.Y + m0 + ym + yk * ldy;
      double* d = As + b * SA + yk * kLdA + ym;
#pragma unroll
      for (int q = 0; q < K / 8; ++q) cp_async16(d + q * 8 * kLdA, g + q * 8 * ldy, 16);
    }
    if (load_x) {
      const double* g = a.X + xk + (n0 + xn) * ldx;
      double* d = Bs + xs * SB + xn * LDB + xk;
#pragma unroll
      for (int q = 0; q < kTN / XROWS; ++q) cp_async16(d + q * XROWS * LDB, g + q * XROWS * ldx, 16);
    }
    {
      const double* g = Csrc + m0 + ym + (n0 + yk) * ldcs;
      double* d = Cs + b * SC + yk * kLdC + ym;
#pragma unroll
      for (int q = 0; q < 8; ++q) cp_async16(d + q * 8 * kLdC, g + q * 8 * ldcs, 16);
    }
    cp_async_commit();
  };
  auto load_edge = [&](int64_t t, int b, int xs, bool load_x) {
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    for (int e = tid; e < K * kTM; e += kRuThreads) {
      const int k = e / kTM, i = e % kTM;
      const bool ok = m0 + i < M;
      cp_async8(As + b * SA + k * kLdA + i, ok ? a.Y + m0 + i + k * ldy : a.Y, ok);
    }
    if (load_x)
      for (int e = tid; e < kTN * K; e += kRuThreads) {
        const int n = e / K, k = e % K;
        const bool ok = n0 + n < N;
        cp_async8(Bs + xs * SB + n * LDB + k, ok ? a.X + k + (n0 + n) * ldx : a.X, ok);
      }
    for (int e = tid; e < kTN * kTM; e += kRuThreads) {
      const int n = e / kTM, i = e % kTM;
      const bool ok = m0 + i < M && n0 + n < N;
      cp_async8(Cs + b * SC + n * kLdC + i, ok ? Csrc + m0 + i + (n0 + n) * ldcs : Csrc, ok);
    }
    cp_async_commit();
  };
  auto full_tile = [&](int64_t t) {
    return ((t % tm) + 1) * kTM <= M && ((t / tm) + 1) * kTN <= N;
  };
  auto load_tile = [&](int64_t t, int b, int xs, bool load_x) {
    if (full_tile(t)) load_full(t, b, xs, load_x);
    else load_edge(t, b, xs, load_x);
  };

  int xs = 0;
  if (t_lo < t_hi) load_tile(t_lo, 0, 0, true);
  int buf = 0;
  for (int64_t t = t_lo; t < t_hi; ++t, buf ^= 1) {
    int xs_next = xs;
    if (t + 1 < t_hi) {
      const bool newx = (t + 1) / tm != t / tm;
      if (newx) xs_next = xs ^ 1;
      load_tile(t + 1, buf ^ 1, xs_next, newx);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As + buf * SA + wm0 + fr;
    const double* bs = Bs + xs * SB + (wn0 + fr) * LDB;
    const double* cs = Cs + buf * SC;
    double acc[4][2][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    double af[2][4], bf[2][2];   // double-buffered fragments (see gemm.cuh)
    auto ldfrag = [&](int buf, int k4) {
#pragma unroll
      for (int x = 0; x < 4; ++x) af[buf][x] = as[(k4 + fk) * kLdA + x * 8];
#pragma unroll
      for (int y = 0; y < 2; ++y) bf[buf][y] = bs[y * 8 * LDB + k4 + fk];
    };
    ldfrag(0, 0);
#pragma unroll
    for (int ks = 0; ks < K / 4; ++ks) {
      if (ks + 1 < K / 4) ldfrag((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) dmma884(acc[x][y], af[ks & 1][x], bf[ks & 1][y]);
    }
    // epilogue: C - acc (C from shared memory; separate subtraction, numpy's C - Y @ X)
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    if (full_tile(t)) {
      double* ct = a.C + (m0 + wm0 + fr) + (n0 + wn0 + 2 * fk) * ldc;
      const double* cst = cs + (wn0 + 2 * fk) * kLdC + wm0 + fr;
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            ct[x * 8 + (y * 8 + e) * ldc] =
                __dsub_rn(cst[(y * 8 + e) * kLdC + x * 8], acc[x][y][e]);
    } else {
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int i = wm0 + x * 8 + fr;
        const int64_t gi = m0 + i;
        if (gi >= M) continue;
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = wn0 + y * 8 + 2 * fk + e;
            const int64_t gj = n0 + j;
            if (gj < N) a.C[gi + gj * ldc] = __dsub_rn(cs[j * kLdC + i], acc[x][y][e]);
          }
      }
    }
    if (a.extra_rows > 0 && (t % tm) == tm - 1) {   // pass-through rows below the update
      for (int e = tid; e < a.extra_rows * kTN; e += kRuThreads) {
        const int r = e % a.extra_rows, j = e / a.extra_rows;
        if (n0 + j < N) a.C[M + r + (n0 + j) * ldc] = Csrc[M + r + (n0 + j) * ldcs];
      }
    }
    __syncthreads();  // buffers `buf` / X slot reloaded by the next prefetch
    xs = xs_next;
  }
}

template <int K>
void launch_rank_update_k(Handle& h, const RuArgs& a, int grid, cudaStream_t s) {
  constexpr size_t smem = (size_t)2 * (K * kLdA + kTN * (K + 4) + kTN * kLdC) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    RQ_CUDA(cudaFuncSetAttribute(rank_update_k_kernel<K>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  rank_update_k_kernel<K><<<grid, kRuThreads, smem, s>>>(a);
}

}  // namespace

bool rank_update(Handle& h, int64_t M, int64_t N, int64_t K, const double* Y, int64_t ldy,
                 const double* X, int64_t ldx, double* C, int64_t ldc, cudaStream_t s,
                 const Status* st, int cat, int max_ctas, Status* snap, const double* Csrc,
                 int64_t ldcs, int extra_rows) {
  if (K < 4 || K > kKMax || (K % 4) != 0 || M <= 0 || N <= 0) return false;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA(cudaFuncSetAttribute(rank_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kRuSmem));
    attr = true;
  }
  const auto al = [](const double* p, int64_t ld) { return ((uintptr_t)p & 15) == 0 && ld % 2 == 0; };
  RuArgs a{M, N, (int)K, Y, ldy, X, ldx, C, ldc, st,
           (h.gemm_vec16 && al(Y, ldy) && al(X, ldx) && al(C, ldc) &&
            (Csrc == nullptr || al(Csrc, ldcs))) ? 1 : 0,
           snap, Csrc, ldcs, extra_rows};
  if (Csrc != nullptr && !(a.vec16 && (K == 32 || K == 64))) return false;   // k-kernel only
  const int64_t ntiles = ((M + kTM - 1) / kTM) * ((N + kTN - 1) / kTN);
  const int cap = max_ctas > 0 ? std::min(max_ctas, h.num_sms) : h.num_sms;
  const int grid = (int)std::min<int64_t>(cap, ntiles);
  ProfScope prof(h, cat, 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + 2.0 * M * N), s);
  if (a.vec16 && K == 64) launch_rank_update_k<64>(h, a, grid, s);
  else if (a.vec16 && K == 32) launch_rank_update_k<32>(h, a, grid, s);
  else rank_update_kernel<<<grid, kRuThreads, kRuSmem, s>>>(a);
  RQ_CHECK_LAUNCH();
  count_launch();
  return true;
}

}  // namespace rq
