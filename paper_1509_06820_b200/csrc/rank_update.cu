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
  unsigned ru_skew_ns;
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

// Two CTAs per SM, single-buffered (104 KB each at K = 64): one CTA's loads,
// epilogue and barriers overlap the other's DMMAs, which the one-CTA
// double-buffered kernel above leaves to the tensor pipe's idle time (ncu:
// DMMA sub-pipe 56% active, barrier + long-scoreboard stalls between tiles).
// The next tile's Y/X are issued before this tile's epilogue (which reads
// only the C buffer) and its C right after.
template <int K>
__global__ void __launch_bounds__(kRuThreads, 2) rank_update_k2_kernel(RuArgs a) {
  snapshot_abort(a);
  if (aborted(a.st)) return;
  constexpr int LDB = K + 4;
  constexpr int SA = K * kLdA, SB = kTN * LDB;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = As + SA;
  double* Cs = Bs + SB;
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
  constexpr int XPER = K / 2, XROWS = kRuThreads / XPER;
  const int ym = 2 * (tid & 31), yk = tid >> 5;
  const int xk = 2 * (tid % XPER), xn = tid / XPER;
  auto full_tile = [&](int64_t t) {
    return ((t % tm) + 1) * kTM <= M && ((t / tm) + 1) * kTN <= N;
  };
  auto load_yx = [&](int64_t t, bool load_x) {
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    if (full_tile(t)) {
      const double* g = a.Y + m0 + ym + yk * ldy;
      double* d = As + yk * kLdA + ym;
#pragma unroll
      for (int q = 0; q < K / 8; ++q) cp_async16(d + q * 8 * kLdA, g + q * 8 * ldy, 16);
      if (load_x) {
        const double* gx = a.X + xk + (n0 + xn) * ldx;
        double* dx = Bs + xn * LDB + xk;
#pragma unroll
        for (int q = 0; q < kTN / XROWS; ++q) cp_async16(dx + q * XROWS * LDB, gx + q * XROWS * ldx, 16);
      }
    } else {
      for (int e = tid; e < K * kTM; e += kRuThreads) {
        const int k = e / kTM, i = e % kTM;
        const bool ok = m0 + i < M;
        cp_async8(As + k * kLdA + i, ok ? a.Y + m0 + i + k * ldy : a.Y, ok);
      }
      if (load_x)
        for (int e = tid; e < kTN * K; e += kRuThreads) {
          const int n = e / K, k = e % K;
          const bool ok = n0 + n < N;
          cp_async8(Bs + n * LDB + k, ok ? a.X + k + (n0 + n) * ldx : a.X, ok);
        }
    }
    cp_async_commit();
  };
  auto load_c = [&](int64_t t) {
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    if (full_tile(t)) {
      const double* g = Csrc + m0 + ym + (n0 + yk) * ldcs;
      double* d = Cs + yk * kLdC + ym;
#pragma unroll
      for (int q = 0; q < 8; ++q) cp_async16(d + q * 8 * kLdC, g + q * 8 * ldcs, 16);
    } else {
      for (int e = tid; e < kTN * kTM; e += kRuThreads) {
        const int n = e / kTM, i = e % kTM;
        const bool ok = m0 + i < M && n0 + n < N;
        cp_async8(Cs + n * kLdC + i, ok ? Csrc + m0 + i + (n0 + n) * ldcs : Csrc, ok);
      }
    }
    cp_async_commit();
  };

  if (t_lo < t_hi) {
    load_yx(t_lo, true);
    load_c(t_lo);
  }
  // the CTAs sharing an SM start together and would stay in phase (both in
  // their epilogue at once): the second wave starts half a tile later
  if (blockIdx.x >= gridDim.x / 2 && a.ru_skew_ns > 0) __nanosleep(a.ru_skew_ns);
  for (int64_t t = t_lo; t < t_hi; ++t) {
    cp_async_wait<0>();
    __syncthreads();
    const double* as = As + wm0 + fr;
    const double* bs = Bs + (wn0 + fr) * LDB;
    double acc[4][2][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    double af[2][4], bf[2][2];
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
    __syncthreads();   // As / Bs consumed
    const bool more = t + 1 < t_hi;
    if (more) load_yx(t + 1, (t + 1) / tm != t / tm);
    const int64_t m0 = (t % tm) * kTM, n0 = (t / tm) * kTN;
    if (full_tile(t)) {
      double* ct = a.C + (m0 + wm0 + fr) + (n0 + wn0 + 2 * fk) * ldc;
      const double* cst = Cs + (wn0 + 2 * fk) * kLdC + wm0 + fr;
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
            if (gj < N) a.C[gi + gj * ldc] = __dsub_rn(Cs[j * kLdC + i], acc[x][y][e]);
          }
      }
    }
    if (a.extra_rows > 0 && (t % tm) == tm - 1) {   // pass-through rows below the update
      for (int e = tid; e < a.extra_rows * kTN; e += kRuThreads) {
        const int r = e % a.extra_rows, j = e / a.extra_rows;
        if (n0 + j < N) a.C[M + r + (n0 + j) * ldc] = Csrc[M + r + (n0 + j) * ldcs];
      }
    }
    __syncthreads();   // Cs consumed
    if (more) load_c(t + 1);
  }
}

template <int K>
void launch_rank_update_k2(Handle& h, const RuArgs& a, int grid, cudaStream_t s) {
  constexpr size_t smem = (size_t)(K * kLdA + kTN * (K + 4) + kTN * kLdC) * sizeof(double);
  kernel_attr((const void*)rank_update_k2_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)smem);
  rank_update_k2_kernel<K><<<grid, kRuThreads, smem, s>>>(a);
}

// Large trailing updates: 128 x 64 tiles ordered n-fastest (a CTA's Y block
// stays resident; only the 32 KB X tile is staged per tile), a 32 x 32 tile
// per warp (16 accumulators, half the fragment loads per DMMA of the 32 x 16
// layout), computed transposed (D = X^T Y^T) so each thread's accumulator
// pair is two consecutive rows of one C column.  Each thread stages exactly
// the C values it will update (16 x 16-byte cp.async into a slot-major
// private area: no barrier, conflict-free reads) at the start of the tile;
// the DMMA loop hides the HBM round trip.  One barrier per tile.
constexpr int kBM = 128, kBN = 64;
// Software pipeline across tiles: the epilogue of tile t - 1 (C - acc from
// the staged C values, 16-byte stores) is interleaved with the first k-steps
// of tile t's DMMAs (two accumulator sets, ping-pong by an unrolled pair of
// steps), and tile t's own C values are staged right after that epilogue has
// consumed the buffer, so the tensor pipe never waits for an epilogue.
template <int K>
__global__ void __launch_bounds__(kRuThreads, 1) rank_update_big_kernel(RuArgs a) {
  snapshot_abort(a);
  if (aborted(a.st)) return;
  constexpr int LDA = kBM + 4;   // As[k][m]   (Y, single buffer)
  constexpr int LDB = K + 4;     // Bs[n][k]   (X, double buffer)
  constexpr int SA = K * LDA, SB = kBN * LDB;
  constexpr int KS = K / 4;      // k-steps per tile
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = As + SA;                                   // [2][SB]
  double2* Cs = reinterpret_cast<double2*>(Bs + 2 * SB);  // [16][kRuThreads]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp & 3) * 32, wn0 = (warp >> 2) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t M = a.M, N = a.N, ldy = a.ldy, ldx = a.ldx, ldc = a.ldc;
  const int64_t tm = (M + kBM - 1) / kBM, tn = (N + kBN - 1) / kBN;
  const int64_t ntiles = tm * tn;
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x;
  const int64_t t_hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  auto load_y = [&](int64_t mb) {   // As[k][m] <- Y[mb*128 + m, k]
    const int64_t m0 = mb * kBM;
    const int64_t mlim = M - m0;
#pragma unroll
    for (int q = 0; q < K * kBM / 2 / kRuThreads; ++q) {
      const int e = tid + q * kRuThreads;
      const int k = e / (kBM / 2), m = 2 * (e % (kBM / 2));
      const int valid = m + 1 < mlim ? 16 : (m < mlim ? 8 : 0);
      cp_async16(As + k * LDA + m, valid ? a.Y + m0 + m + k * ldy : a.Y, valid);
    }
  };
  auto load_x = [&](int64_t nb, int b) {   // Bs[b][n][k] <- X[k, nb*64 + n]
    const int64_t n0 = nb * kBN;
#pragma unroll
    for (int q = 0; q < kBN * K / 2 / kRuThreads; ++q) {
      const int e = tid + q * kRuThreads;
      const int n = e / (K / 2), k = 2 * (e % (K / 2));
      const int valid = n0 + n < N ? 16 : 0;
      cp_async16(Bs + b * SB + n * LDB + k, valid ? a.X + k + (n0 + n) * ldx : a.X, valid);
    }
  };
  // my C values of tile t (transposed mapping: D = X^T Y^T, so the pair is
  // rows mt0 + 8y, +1 of column nt0 + 8x)
  auto tile_c0 = [&](int64_t t, int64_t& mt0, int64_t& nt0, bool& full) {
    const int64_t mb = t / tn, nb = t % tn;
    mt0 = mb * kBM + wm0 + 2 * fk;
    nt0 = nb * kBN + wn0 + fr;
    full = (mb + 1) * kBM <= M && (nb + 1) * kBN <= N;
  };
  auto stage_c = [&](int64_t t) {
    int64_t mt0, nt0;
    bool full;
    tile_c0(t, mt0, nt0, full);
    const double* cp = a.C + mt0 + nt0 * ldc;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int64_t gi = mt0 + y * 8, gj = nt0 + x * 8;
        const int valid = full ? 16 : (gj < N ? (gi + 1 < M ? 16 : (gi < M ? 8 : 0)) : 0);
        cp_async16(Cs + (x * 4 + y) * kRuThreads + tid, valid ? cp + y * 8 + x * 8 * ldc : a.C,
                   valid);
      }
    cp_async_commit();
  };
  // C - acc for the (x, y) pair `q` of tile t (separate subtraction, numpy's C - Y @ X)
  auto epi = [&](const double (&acc)[4][4][2], int64_t t, int q) {
    int64_t mt0, nt0;
    bool full;
    tile_c0(t, mt0, nt0, full);
    const int x = q >> 2, y = q & 3;
    const double2 c = Cs[q * kRuThreads + tid];
    double2 r;
    r.x = __dsub_rn(c.x, acc[x][y][0]);
    r.y = __dsub_rn(c.y, acc[x][y][1]);
    const int64_t gi = mt0 + y * 8, gj = nt0 + x * 8;
    if (full) {
      __stcg(reinterpret_cast<double2*>(a.C + gi + gj * ldc), r);
    } else if (gj < N) {
      if (gi < M) a.C[gi + gj * ldc] = r.x;
      if (gi + 1 < M) a.C[gi + 1 + gj * ldc] = r.y;
    }
  };
  if (t_lo >= t_hi) return;
  int xb = 0;
  bool ywait = true;   // the next step must also wait for a Y block
  load_y(t_lo / tn);
  load_x(t_lo % tn, 0);
  cp_async_commit();
  // one tile: its DMMAs into `cur`, the previous tile's epilogue from `prev`
  auto step = [&](double (&cur)[4][4][2], const double (&prev)[4][4][2], int64_t t) {
    const bool has_prev = t > t_lo;
    // groups in flight: X(t) [+ Y], then C(t - 1)
    if (ywait || !has_prev) cp_async_wait<0>();
    else cp_async_wait<1>();
    __syncthreads();   // tile t's operands visible; everyone is done with tile t - 1's X buffer
    ywait = false;
    const bool more = t + 1 < t_hi;
    if (more) {
      load_x((t + 1) % tn, xb ^ 1);
      cp_async_commit();
    }
    if (!has_prev) stage_c(t);
    const double* xs_ = Bs + xb * SB + (wn0 + fr) * LDB;   // A fragment: X[k][n]
    const double* ys_ = As + wm0 + fr;                      // B fragment: Y[m][k]
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) cur[x][y][0] = cur[x][y][1] = 0.0;
    double af[2][4], bf[2][4];
    auto ldfrag = [&](int fb, int k4) {
#pragma unroll
      for (int x = 0; x < 4; ++x) af[fb][x] = xs_[x * 8 * LDB + k4 + fk];
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[fb][y] = ys_[(k4 + fk) * LDA + y * 8];
    };
    ldfrag(0, 0);
    if (has_prev) {
      if (more) cp_async_wait<1>();   // C(t - 1) (X(t + 1) may still fly)
      else cp_async_wait<0>();
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (ks + 1 < KS) ldfrag((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma884(cur[x][y], af[ks & 1][x], bf[ks & 1][y]);
      // previous tile's epilogue spread over the first k-steps
      if (has_prev && ks < 8) {
        epi(prev, t - 1, 2 * ks);
        epi(prev, t - 1, 2 * ks + 1);
      }
      if (KS > 8 && has_prev && ks == 8) stage_c(t);   // own slots, after their last read
    }
    // K = 32 (8 k-steps): the epilogue took every step, stage after the loop
    if (KS <= 8 && has_prev) stage_c(t);
    if (more && (t + 1) / tn != t / tn) {   // next tile starts a new Y block
      __syncthreads();
      load_y((t + 1) / tn);
      cp_async_commit();
      ywait = true;
    }
    xb ^= 1;
  };
  double accA[4][4][2], accB[4][4][2];
  int64_t t = t_lo;
  for (; t + 1 < t_hi; t += 2) {
    step(accA, accB, t);
    step(accB, accA, t + 1);
  }
  if (t < t_hi) {
    step(accA, accB, t);
    cp_async_wait<0>();
#pragma unroll
    for (int q = 0; q < 16; ++q) epi(accA, t, q);
  } else {
    cp_async_wait<0>();
#pragma unroll
    for (int q = 0; q < 16; ++q) epi(accB, t - 1, q);
  }
}

template <int K>
void launch_rank_update_big(Handle& h, const RuArgs& a, int grid, cudaStream_t s) {
  constexpr size_t smem =
      ((size_t)K * (kBM + 4) + 2 * (size_t)kBN * (K + 4)) * sizeof(double) + 16 * kRuThreads * 16;
      kernel_attr((const void*)rank_update_big_kernel<K>,
                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rank_update_big_kernel<K><<<grid, kRuThreads, smem, s>>>(a);
}

template <int K>
void launch_rank_update_k(Handle& h, const RuArgs& a, int grid, cudaStream_t s) {
  constexpr size_t smem = (size_t)2 * (K * kLdA + kTN * (K + 4) + kTN * kLdC) * sizeof(double);
  kernel_attr((const void*)rank_update_k_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)smem);
  rank_update_k_kernel<K><<<grid, kRuThreads, smem, s>>>(a);
}

}  // namespace

bool rank_update(Handle& h, int64_t M, int64_t N, int64_t K, const double* Y, int64_t ldy,
                 const double* X, int64_t ldx, double* C, int64_t ldc, cudaStream_t s,
                 const Status* st, int cat, int max_ctas, Status* snap, const double* Csrc,
                 int64_t ldcs, int extra_rows) {
  if (K < 4 || (K > kKMax && K != 128) || (K % 4) != 0 || M <= 0 || N <= 0) return false;
  // the TMA-fed grouped kernel (rank_update_tma.cu) for K in {32, 64, 128}
  if (Csrc == nullptr && extra_rows == 0 &&
      rank_update_tma(h, M, N, K, Y, ldy, X, ldx, C, ldc, s, st, cat, max_ctas, snap))
    return true;
  kernel_attr((const void*)rank_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)kRuSmem);
  const auto al = [](const double* p, int64_t ld) { return ((uintptr_t)p & 15) == 0 && ld % 2 == 0; };
  RuArgs a{M, N, (int)K, Y, ldy, X, ldx, C, ldc, st,
           (h.gemm_vec16 && al(Y, ldy) && al(X, ldx) && al(C, ldc) &&
            (Csrc == nullptr || al(Csrc, ldcs))) ? 1 : 0,
           snap, Csrc, ldcs, extra_rows, (unsigned)h.ru_skew_ns};
  if (Csrc != nullptr && !(a.vec16 && (K == 32 || K == 64))) return false;   // k-kernel only
  if (K == 128 && !(h.ru_big && a.vec16 && Csrc == nullptr && extra_rows == 0 && M >= kBM))
    return false;   // the caller's generic GEMM
  const int64_t ntiles = ((M + kTM - 1) / kTM) * ((N + kTN - 1) / kTN);
  const int cap = max_ctas > 0 ? std::min(max_ctas, h.num_sms) : h.num_sms;
  const int grid = (int)std::min<int64_t>(cap, ntiles);
  ProfScope prof(h, cat, 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + 2.0 * M * N), s);
  if (h.ru_big && a.vec16 && (K == 64 || K == 32 || K == 128) && Csrc == nullptr &&
      extra_rows == 0 && M >= kBM) {
    const int64_t tiles = ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
    const int gridb = (int)std::min<int64_t>(cap, tiles);
    if (K == 64) launch_rank_update_big<64>(h, a, gridb, s);
    else if (K == 32) launch_rank_update_big<32>(h, a, gridb, s);
    else {
      // K = 128 (b = 128, cfg5): two K = 64 passes, C -= Y[:, :64] X[:64] then
      // C -= Y[:, 64:] X[64:] (twice the C traffic, but the 64-deep tiles
      // run at ~24 TF/s against ~15 for a generic 128-deep GEMM)
      RuArgs a2 = a;
      a2.K = 64;
      launch_rank_update_big<64>(h, a2, gridb, s);
      RQ_CHECK_LAUNCH();
      count_launch();
      a2.Y = Y + 64 * ldy;
      a2.X = X + 64;
      a2.snap = nullptr;
      launch_rank_update_big<64>(h, a2, gridb, s);
    }
  } else if (h.ru_two_ctas && a.vec16 && (K == 64 || K == 32)) {
    const int grid2 = (int)std::min<int64_t>(2 * cap, ntiles);
    if (K == 64) launch_rank_update_k2<64>(h, a, grid2, s);
    else launch_rank_update_k2<32>(h, a, grid2, s);
  } else if (a.vec16 && K == 64) launch_rank_update_k<64>(h, a, grid, s);
  else if (a.vec16 && K == 32) launch_rank_update_k<32>(h, a, grid, s);
  else rank_update_kernel<<<grid, kRuThreads, kRuSmem, s>>>(a);
  RQ_CHECK_LAUNCH();
  count_launch();
  return true;
}

}  // namespace rq
