// K5b: communication-avoiding panel QR -- CholeskyQR2 for R, then the
// Householder vectors reconstructed from the orthonormal factor (Ballard et
// al., "Reconstructing Householder vectors from TSQR").  Same outputs as the
// column-by-column panel kernel (panel.cu: R in the panel rows, unit-lower
// Y, tau; qrcp.py:206-219 panel_householder), but with 6 grid barriers per
// panel instead of one exchange per column.
//
// Why it reproduces the reference's reflectors: the Householder QR of a full
// column-rank panel P is unique up to the row signs of R.  With the
// reference's convention beta = -sign(alpha)||x|| (kernels.py:26-44) the
// compact-WY form satisfies  Q~ S - [I; 0] = Y (-T Y1^T),  i.e. the LU
// factorisation (no pivoting) of Q~ S - [I; 0] has L = Y and U = -T Y1^T,
// where Q~ is any orthonormal basis with P = Q~ R~ and S the diagonal sign
// matrix making R = S R~.  Choosing s_j = -sign(c_j) for the eliminated
// diagonal c_j gives u_jj = -(1 + |c_j|) = -tau_j with tau_j in [1, 2], which
// is exactly the reference's tau = (beta - alpha) / beta.
//
//   G1 = P^T P                       all CTAs (DMMA partials) + fixed-order reduction
//   R1 = chol(G1), R1^{-1}           CTA 0
//   G2 = (P R1^{-1})^T (P R1^{-1})   all CTAs
//   R2 = I + F  (F = triu(G2 - I), diagonal halved; exact to O(|G2 - I|^2)
//               because |G2 - I| <= 1e-10 is required)
//   R~ = R2 R1,  Q~_top = P_top R1^{-1} (I - F),  LU with signs -> S, U, Y_top   CTA 0
//   M = R1^{-1} (I - F) S U^{-1} (CTA 0)  |  sample update's S11 R1^{-1} (I - F) S
//   (CTA 1)  |  T = -U Y1^{-T}, A1 = Y1 T, A2 = -R1^{-1} (I - F) S Y1^{-T} (CTA 2)
//   Y_below = P_below M                            all CTAs
//
// The fast path only commits when it is safe to skip the reference's
// column-by-column arithmetic: Cholesky succeeds, diag-ratio of R1 <= 1e3,
// |G2 - I| <= 1e-10, and every |R_jj| clears both the _panel_rank threshold
// (randomized.py:150-155) and the sample-update degenerate threshold
// (randomized.py:117) by a relative margin.  Otherwise nothing is written,
// *fast_ok = 0, and the exact kernel that follows on the stream runs.
#include "gemm.cuh"
#include "runtime.hpp"
#include "tri.cuh"

namespace rq {

namespace {

constexpr int kFT = 256;            // threads per CTA
constexpr int kFMaxBw = 64;
constexpr int kFRows = 64;          // panel rows per chunk
constexpr double kFastMaxKappa = 1e3;
constexpr double kFastMaxE = 1e-10;
constexpr double kFastMargin = 1.0 + 1e-6;

struct FastArgs {
  int64_t mm;
  int n, n8, ld;                    // panel width, padded width, smem row stride
  const double* P; int64_t ldp;
  double* Rdst; int64_t ldr; int64_t rrows;
  double* Y; int64_t ldy;
  double* tau;
  double* T; int64_t ldt;           // optional T factor (nullptr: not wanted)
  double tol, guard;                // < 0: no threshold
  int abort_on_decline;             // speculative driver: decline -> Status.abort (kAbortPanelFast)
  int defer_zero;                   // leave the panel rows below the diagonal to the caller
  const double* S11; int64_t lds11; // optional: sample block for the sample update's M
  double* msu;                      // out (if S11): M = S11 R11^{-1}, b x b column-major
  double* a12;                      // out (if T): A1 = Y1 T, A2 = M T, b x b column-major each
  int64_t l2_extra;                 // extra level-2 count on commit (second half of a wider panel)
  int degen_commit;                 // commit a clearly degenerate R11 (Status.degenerate = 1)
  int usable_total;                 // Status.usable on commit (0: the panel width)
  int64_t i0;
  int64_t nchunks;
  Status* st;
  unsigned int* bar;                // [0] barrier, [1] exit count, [2] fail, [4] skip flag
  double* gpart;                    // [Q][n8*n8]
  double* gmat;                     // [5][n8*n8]: G1, R1, R1^{-1}, G2, M
  double* gx;                       // [2][n8*n8] + [n8]: L, U, signs (CTA 0 -> the stage-2 helpers)
  long long* dbg;
};

RQ_DEV double ldcg(const double* p) { return __ldcg(p); }

// rows [ch*64, ch*64+64) x cols [0, n8) of the column-major panel into a
// row-major chunk (zero padded), in two halves so the next chunk's global
// loads (load_regs) are in flight while the current chunk is multiplied
RQ_DEV void load_regs(const FastArgs& a, int64_t ch, double (&v)[16]) {
  const int64_t r0 = ch * kFRows;
  const int r = threadIdx.x & (kFRows - 1), c0 = threadIdx.x / kFRows;  // 4 columns per pass
  const int64_t gr = r0 + r;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = c0 + 4 * k;
    v[k] = (c < a.n && gr < a.mm) ? a.P[gr + (int64_t)c * a.ldp] : 0.0;
  }
}
RQ_DEV void store_regs(const FastArgs& a, const double (&v)[16], double* C) {
  const int r = threadIdx.x & (kFRows - 1), c0 = threadIdx.x / kFRows;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = c0 + 4 * k;
    if (c < a.n8) C[r * a.ld + c] = v[k];
  }
}

// Out(rows x n8) = A(rows x n8) B(n8 x n8), all row-major with stride ld;
// warp w owns rows [8w, 8w+8).  kUA / kUB: A / B upper triangular (their zero
// k-ranges are skipped; FP64 DMMA is ~4 cycles per 8x8x4 per SM, so a full
// 64^3 product is ~4K cycles and triangular structure matters).
template <bool kUA, bool kUB>
RQ_DEV void chunk_mm(const double* A, const double* B, double* Out, int rows, int n8, int ld) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (8 * warp >= rows) return;
  const int fr = lane >> 2, fk = lane & 3;
  const int nt = n8 / 8;
  double acc[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
  for (int k4 = kUA ? 8 * warp : 0; k4 < n8; k4 += 4) {
    const double av = A[(8 * warp + fr) * ld + k4 + fk];
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (t < nt && (!kUB || k4 < 8 * (t + 1))) dmma884(acc[t], av, B[(k4 + fk) * ld + t * 8 + fr]);
  }
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (t < nt) {
      Out[(8 * warp + fr) * ld + t * 8 + 2 * fk] = acc[t][0];
      Out[(8 * warp + fr) * ld + t * 8 + 2 * fk + 1] = acc[t][1];
    }
}

// acc += C^T C over the 64 chunk rows, upper 8x8 tiles only; warp w owns
// tiles w, w+8, ... of the row-wise upper tile list
RQ_DEV void tile_of(int t, int nt, int& ti, int& tj) {
  ti = 0;
  while (t >= nt - ti) { t -= nt - ti; ++ti; }
  tj = ti + t;
}
RQ_DEV void chunk_gram(const double* C, int n8, int ld, double (&acc)[5][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fk = lane & 3;
  const int nt = n8 / 8, ntiles = nt * (nt + 1) / 2;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int t = warp + 8 * q;
    if (t < ntiles) {
      int ti, tj;
      tile_of(t, nt, ti, tj);
      for (int k4 = 0; k4 < kFRows; k4 += 4)
        dmma884(acc[q], C[(k4 + fk) * ld + ti * 8 + fr], C[(k4 + fk) * ld + tj * 8 + fr]);
    }
  }
}
RQ_DEV void store_gram(double* dst, int n8, const double (&acc)[5][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fk = lane & 3;
  const int nt = n8 / 8, ntiles = nt * (nt + 1) / 2;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int t = warp + 8 * q;
    if (t < ntiles) {
      int ti, tj;
      tile_of(t, nt, ti, tj);
      dst[(ti * 8 + fr) * n8 + tj * 8 + 2 * fk] = acc[q][0];
      dst[(ti * 8 + fr) * n8 + tj * 8 + 2 * fk + 1] = acc[q][1];
    }
  }
}

// element / row of a 4-wide register array for a warp-uniform index, as a
// uniform branch (compare-select chains cost ~40% of the LU's issue slots)
RQ_DEV double pick4(const double (&v)[4], int i) {
  switch (i) {
    case 1: return v[1];
    case 2: return v[2];
    case 3: return v[3];
    default: return v[0];
  }
}
RQ_DEV void pick_row4(const double (&m)[4][4], int c, double (&out)[4]) {
  switch (c) {
    case 1:
#pragma unroll
      for (int b = 0; b < 4; ++b) out[b] = m[1][b];
      break;
    case 2:
#pragma unroll
      for (int b = 0; b < 4; ++b) out[b] = m[2][b];
      break;
    case 3:
#pragma unroll
      for (int b = 0; b < 4; ++b) out[b] = m[3][b];
      break;
    default:
#pragma unroll
      for (int b = 0; b < 4; ++b) out[b] = m[0][b];
  }
}

__global__ void __launch_bounds__(kFT, 1) panel_fast_kernel(FastArgs a) {
  if (aborted(a.st)) {  // set only by earlier launches: uniform over the grid
    if (blockIdx.x == 0 && threadIdx.x == 0) a.bar[4] = 1;   // nothing downstream runs either
    return;
  }
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_fail, s_degen;
  __shared__ double s_sign[kFMaxBw], s_c[kFMaxBw], s_dinv[kFMaxBw];
  auto lane_of = [](int t) { return t & 31; };
  const int tid = threadIdx.x;
  const int me = blockIdx.x, Q = gridDim.x;
  const int n = a.n, n8 = a.n8, ld = a.ld;
  const int lg8 = n8 == 64 ? 6 : (n8 == 32 ? 5 : (n8 == 16 ? 4 : 3));
  const int nn = n8 * n8;
  const int rstep = kFT >> lg8, r0 = tid >> lg8, c0 = tid & (n8 - 1);  // 2D element loops
  const size_t W = (size_t)kFRows * ld;   // a 64-row chunk or an n8 x n8 matrix
  double* W0 = sm;
  double* W1 = W0 + W;
  double* W2 = W1 + W;
  double* W3 = W2 + W;
  double* W4 = W3 + W;
  double* W5 = W4 + W;
  unsigned int epoch = 0;
  const bool timing = a.dbg != nullptr && me == 0 && tid == 0;
  long long t0 = timing ? clock64() : 0;
  auto mark = [&](int k) {
    if (timing) {
      const long long t1 = clock64();
      a.dbg[8 + k] = t1 - t0;
      t0 = t1;
    }
  };
  long long u0 = timing ? clock64() : 0;
  auto sub = [&](int k) {  // serial-section timers (CTA 0; barrier first so waits are charged here)
    if (a.dbg != nullptr) {
      __syncthreads();
      if (timing) {
        const long long u1 = clock64();
        a.dbg[16 + k] = u1 - u0;
        u0 = u1;
      }
    }
  };
  auto finish = [&]() {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(&a.bar[1], 1u) == (unsigned)Q - 1) {  // everyone is past every barrier
        a.bar[0] = 0;
        a.bar[1] = 0;
      }
    }
  };
  double* red = W5 + W - 8 * 32;   // reduction scratch (end of W5)
  auto reduce = [&](double* dst) {  // dst = sum over CTAs of gpart, fixed order
    const int lane = tid & 31, grp = tid >> 5;
    for (int e0 = me * 32; e0 < nn; e0 += Q * 32) {
      const int e = e0 + lane;
      double sacc = 0.0;
      if (e < nn) {
        double v[16];
        int q = grp;
#pragma unroll
        for (int k = 0; k < 16; ++k, q += 8) v[k] = q < Q ? ldcg(a.gpart + (size_t)q * nn + e) : 0.0;
        for (; q < Q; q += 8) sacc += ldcg(a.gpart + (size_t)q * nn + e);
#pragma unroll
        for (int k = 0; k < 16; ++k) sacc += v[k];
      }
      red[grp * 32 + lane] = sacc;
      __syncthreads();
      if (grp == 0 && e < nn) {
        double t = red[lane];
#pragma unroll
        for (int g = 1; g < 8; ++g) t += red[g * 32 + lane];
        dst[e] = t;
      }
      __syncthreads();
    }
  };
  // with one chunk per CTA the panel rows stay in W0 from phase A to phase C
  // (CTA 0 reuses W0 for its serial sections and reloads)
  const bool resident = a.nchunks <= Q && me != 0;
  double acc[5][2];

  // ---- phase A: partial G1 = P^T P
#pragma unroll
  for (int q = 0; q < 5; ++q) acc[q][0] = acc[q][1] = 0.0;
  double pre[16];   // the next chunk, loaded while the current one is multiplied
  if (me < a.nchunks) load_regs(a, me, pre);
  for (int64_t ch = me; ch < a.nchunks; ch += Q) {
    __syncthreads();
    store_regs(a, pre, W0);
    __syncthreads();
    if (ch + Q < a.nchunks) load_regs(a, ch + Q, pre);
    chunk_gram(W0, n8, ld, acc);
  }
  store_gram(a.gpart + (size_t)me * nn, n8, acc);
  mark(0);
  grid_barrier_patient(&a.bar[0], epoch);
  reduce(a.gmat);
  grid_barrier_patient(&a.bar[0], epoch);
  mark(1);

  // ---- CTA 0: R1 = chol(G1), R1^{-1}
  // elimination steps: thread (ty, tx) keeps elements (ty + 16c, tx + 16b) in
  // registers; the pivot row goes through shared memory, one barrier per step
  const int ty = tid >> 4, tx = tid & 15;
  if (me == 0) {
    double* R1 = W1;
    for (int i = r0; i < n8; i += rstep) R1[i * ld + c0] = (i == c0 && i >= n) ? 1.0 : 0.0;
    double g[4][4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * c, l = tx + 16 * b;
        g[c][b] = (i < n && l < n && i <= l) ? ldcg(a.gmat + i * n8 + l) : 0.0;
      }
    if (tid == 0) s_fail = 0;
    __syncthreads();
    sub(0);
    // two columns per barrier: rows j and j+1 (j even) live in the two
    // halves of one warp, which factors the 2x2 pivot block with shuffles
    for (int j = 0; j < n; j += 2) {
      const int cj = j >> 4, tj = j & 15;
      const bool two = j + 1 < n;
      if ((ty >> 1) == (tj >> 1)) {
        const bool h1 = (ty & 1) != 0;       // lanes 16..31: row j+1
        double gj[4];
        pick_row4(g, cj, gj);
        const double d0 = __shfl_sync(0xffffffffu, pick4(gj, cj), tj);  // G[j][j]
        const double rinv0 = rsqrt(d0);
        double r0v[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) r0v[b] = __shfl_xor_sync(0xffffffffu, gj[b] * rinv0, 16);
        // row j+1 after pivot j: g - R[j][j+1] R[j][l]
        const double rj1 = h1 ? pick4(r0v, cj) : pick4(gj, cj) * rinv0;
        const double r01 = __shfl_sync(0xffffffffu, rj1, tj + 1);       // R[j][j+1]
        double g1[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) g1[b] = __fma_rn(-r01, r0v[b], gj[b]);
        const double d1 = two ? __shfl_sync(0xffffffffu, pick4(g1, cj), 16 + tj + 1) : 1.0;
        const double rinv1 = rsqrt(d1);
        if (!(d0 > 0.0) || !(d1 > 0.0)) {
          if (lane_of(tid) == 0) s_fail = 1;
        } else if (!h1) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int l = tx + 16 * b;
            if (l >= j && l < n) R1[j * ld + l] = (l == j) ? d0 * rinv0 : gj[b] * rinv0;
          }
        } else if (two) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int l = tx + 16 * b;
            if (l >= j + 1 && l < n) R1[(j + 1) * ld + l] = (l == j + 1) ? d1 * rinv1 : g1[b] * rinv1;
          }
        }
      }
      __syncthreads();
      if (s_fail) break;
      // unguarded: rows/columns <= j+1 are dead once published, R1 is zero
      // below the diagonal and in the padding, so only live entries change
      double ri0[4], rl0[4], ri1[4], rl1[4];
      const int j1 = two ? j + 1 : j;   // row j+1 of R1 is zero when absent
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * b, l = tx + 16 * b;
        ri0[b] = R1[j * ld + i];
        rl0[b] = R1[j * ld + l];
        ri1[b] = two ? R1[j1 * ld + i] : 0.0;
        rl1[b] = two ? R1[j1 * ld + l] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          g[c][b] = __fma_rn(-ri1[c], rl1[b], __fma_rn(-ri0[c], rl0[b], g[c][b]));
    }
    __syncthreads();
    if (tid < 32 && !s_fail) {   // diagonal ratio of R1 (lower bound of its condition number)
      double mx = 0.0, mn = 1e300;
      for (int j = tid; j < n; j += 32) {
        const double r = R1[j * ld + j];
        mx = fmax(mx, r);
        mn = fmin(mn, r);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      if (tid == 0 && mx > kFastMaxKappa * mn) s_fail = 1;
    }
    __syncthreads();
    sub(1);
    if (!s_fail) {
      for (int j = tid; j < n8; j += kFT) s_dinv[j] = j < n ? 1.0 / R1[j * ld + j] : 1.0;
      __syncthreads();
      upper_inverse<kFT>(R1, s_dinv, W2, W3, n8, ld);
      __syncthreads();
      sub(2);
      for (int i = r0; i < n8; i += rstep) {
        a.gmat[nn + i * n8 + c0] = R1[i * ld + c0];
        a.gmat[2 * nn + i * n8 + c0] = W2[i * ld + c0];
      }
    }
    if (tid == 0) {
      a.bar[2] = s_fail;
      if (s_fail) {
        a.bar[4] = 0;
        if (a.abort_on_decline) {
          a.st->abort_i0 = a.i0;
          __threadfence();
          a.st->abort = kAbortPanelFast;
        }
      }
    }
    sub(3);
  }
  mark(2);
  grid_barrier_patient(&a.bar[0], epoch);
  if (__ldcg((const int*)&a.bar[2])) {
    finish();
    return;
  }

  // ---- phase B: partial G2 = (P R1^{-1})^T (P R1^{-1})
  for (int i = r0; i < n8; i += rstep) W2[i * ld + c0] = ldcg(a.gmat + 2 * nn + i * n8 + c0);
#pragma unroll
  for (int q = 0; q < 5; ++q) acc[q][0] = acc[q][1] = 0.0;
  if (!resident && me < a.nchunks) load_regs(a, me, pre);
  for (int64_t ch = me; ch < a.nchunks; ch += Q) {
    __syncthreads();
    if (!resident) store_regs(a, pre, W0);
    __syncthreads();
    if (!resident && ch + Q < a.nchunks) load_regs(a, ch + Q, pre);
    chunk_mm<false, true>(W0, W2, W1, kFRows, n8, ld);
    __syncthreads();
    chunk_gram(W1, n8, ld, acc);
  }
  store_gram(a.gpart + (size_t)me * nn, n8, acc);
  mark(3);
  grid_barrier_patient(&a.bar[0], epoch);
  reduce(a.gmat + 3 * nn);
  grid_barrier_patient(&a.bar[0], epoch);
  mark(4);

  // ---- CTA 0: F, R~, LU with signs (stage 1 of the second serial section)
  // Stage 2 (after one more grid barrier) is spread over three CTAs: CTA 0
  // keeps the critical product M = R1^{-1} (I - F) S U^{-1} (phase C needs it),
  // CTA 1 forms the sample update's M, CTA 2 the T factor and block_finish's
  // A1, A2 -- all from L, U and the signs CTA 0 publishes in gx.
  double* gxL = a.gx;                  // L = Y1 (strictly lower part), row-major n8 x n8
  double* gxU = a.gx + nn;             // U, row-major
  double* gxs = a.gx + 2 * nn;         // signs s_j
  double* Mdst = a.gmat + 4 * nn;      // M (gmat[3] keeps G2: the helpers re-form F from it)
  if (me == 0) {
    // CTA 0 factored chunk 0 in phase B: with one chunk per CTA its W1 still
    // holds Q1 rows [0, 64), i.e. Q1_top
    const bool q1top = a.nchunks <= Q;
    double* Rt = W0;   // R~ = (I + F) R1
    double* Q1 = W1;   // Q1_top, then the U rows of the LU
    double* Ri = W2;   // R1^{-1} (from phase B)
    double* F = W3;
    double* R1 = W4;   // R1, then U^{-1} / M'
    double* T5 = W5;   // P_top / products, then L
    if (tid == 0) s_fail = 0;
    __syncthreads();
    for (int i = r0; i < n8; i += rstep) {
      const int l = c0, e = i * n8 + l;
      double f = 0.0;
      if (i <= l && l < n) {
        const double E = ldcg(a.gmat + 3 * nn + e) - (i == l ? 1.0 : 0.0);
        if (!(fabs(E) <= kFastMaxE)) s_fail = 1;
        f = (i == l) ? 0.5 * E : E;
      }
      F[i * ld + l] = f;
      R1[i * ld + l] = ldcg(a.gmat + nn + e);
      if (!q1top) T5[i * ld + l] = (i < n && l < n) ? a.P[i + (int64_t)l * a.ldp] : 0.0;
    }
    __syncthreads();
    sub(4);
    chunk_mm<true, true>(F, R1, Rt, n8, n8, ld);             // F R1
    if (!q1top) chunk_mm<false, true>(T5, Ri, Q1, n8, n8, ld);  // Q1_top = P_top R1^{-1}
    __syncthreads();
    for (int i = r0; i < n8; i += rstep)
      Rt[i * ld + c0] = i <= c0 ? Rt[i * ld + c0] + R1[i * ld + c0] : 0.0;
    chunk_mm<false, true>(Q1, F, T5, n8, n8, ld);            // Q1_top F
    __syncthreads();
    double z[4][4];   // Q~_top = Q1_top (I - F), register-owned for the LU
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * c, l = tx + 16 * b;
        z[c][b] = (i < n && l < n) ? Q1[i * ld + l] - T5[i * ld + l] : 0.0;
      }
    __syncthreads();
    sub(5);
    // LU of Q~_top S - I without pivoting; the sign of column j is chosen at
    // step j, so U is kept unsigned (rows in Q1) and signed afterwards
    for (int j = 0; j < n; ++j) {
      const int cj = j >> 4, tj = j & 15;
      if (ty == tj) {
        double zj[4];
        pick_row4(z, cj, zj);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int l = tx + 16 * b;
          if (l >= j && l < n) Q1[j * ld + l] = zj[b];
        }
      }
      __syncthreads();
      const double piv = Q1[j * ld + j];
      const double sj = piv >= 0.0 ? -1.0 : 1.0;
      const double linv = -sj * __drcp_rn(fabs(piv) + 1.0);
      if (tid == 0) {
        s_sign[j] = sj;
        s_c[j] = piv;
      }
      // unguarded: rows/columns <= j are dead (U rows live in Q1, L in T5),
      // padding rows/columns are exactly zero
      double li[4], zl[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = ty + 16 * c;
        li[c] = __shfl_sync(0xffffffffu, pick4(z[c], cj), tj, 16) * linv;
        if (tx == tj && i > j && i < n) T5[i * ld + j] = li[c];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) zl[b] = Q1[j * ld + tx + 16 * b];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int b = 0; b < 4; ++b) z[c][b] = __fma_rn(-li[c], zl[b], z[c][b]);
    }
    __syncthreads();
    // U = -(1 + |c_j|) on the diagonal, s_l u_jl above it
    for (int i = r0; i < n8; i += rstep) {
      const int l = c0;
      double u = (i == l) ? 1.0 : 0.0;
      if (l < n && i <= l) u = (i == l) ? -(fabs(s_c[i]) + 1.0) : s_sign[l] * Q1[i * ld + l];
      Q1[i * ld + l] = u;
    }
    if (tid == 0) s_degen = 0;
    __syncthreads();
    for (int j = tid; j < n; j += kFT) {
      s_dinv[j] = -__drcp_rn(fabs(s_c[j]) + 1.0);
      const double rjj = fabs(Rt[j * ld + j]);
      if (a.tol >= 0.0 && !(rjj > kFastMargin * a.tol)) s_fail = 1;
      if (a.guard >= 0.0 && !(rjj > kFastMargin * a.guard)) {
        // below the sample update's degenerate guard (randomized.py:117):
        // committable only when clearly below (the verdict cannot flip)
        if (a.degen_commit && rjj * kFastMargin < a.guard) s_degen = 1;
        else s_fail = 1;
      }
    }
    for (int j = n + tid; j < n8; j += kFT) s_dinv[j] = 1.0;
    __syncthreads();
    if (!s_fail) {
      for (int i = r0; i < n8; i += rstep) {
        gxL[i * n8 + c0] = (i > c0 && i < n) ? T5[i * ld + c0] : 0.0;
        gxU[i * n8 + c0] = Q1[i * ld + c0];
      }
      for (int j = tid; j < n8; j += kFT) gxs[j] = j < n ? s_sign[j] : 1.0;
    }
    if (tid == 0) {
      a.bar[2] = s_fail;
      a.bar[4] = s_fail ? 0 : 1;
      if (s_fail && a.abort_on_decline) {
        a.st->abort_i0 = a.i0;
        __threadfence();
        a.st->abort = kAbortPanelFast;
      }
    }
    sub(6);
  }
  mark(5);
  grid_barrier_patient(&a.bar[0], epoch);
  if (__ldcg((const int*)&a.bar[2])) {
    finish();
    return;
  }

  // ---- stage 2: CTA 0 -> M and the top rows; CTA 1 -> sample update's M; CTA 2 -> T, A1, A2
  bool arrived = false;
  if (me == 0) {
    double* Rt = W0;
    double* Q1 = W1;   // U
    double* Ri = W2;
    double* F = W3;
    double* R1 = W4;   // U^{-1}, V, M'
    double* T5 = W5;   // L, then scratch
    // Y_top = L before T5 becomes scratch
    for (int e = tid; e < n * n; e += kFT) {
      const int l = e / n, i = e - l * n;
      a.Y[i + (int64_t)l * a.ldy] = i < l ? 0.0 : (i == l ? 1.0 : T5[i * ld + l]);
    }
    __syncthreads();
    upper_inverse<kFT>(Q1, s_dinv, R1, T5, n8, ld);   // U^{-1}
    __syncthreads();
    sub(7);
    for (int i = r0; i < n; i += rstep) R1[i * ld + c0] *= s_sign[i];   // V = S U^{-1}
    __syncthreads();
    chunk_mm<true, true>(F, R1, T5, n8, n8, ld);   // F V
    __syncthreads();
    for (int i = r0; i < n8; i += rstep) R1[i * ld + c0] -= T5[i * ld + c0];   // M' = (I - F) V
    __syncthreads();
    chunk_mm<true, true>(Ri, R1, T5, n8, n8, ld);  // M = R1^{-1} M'
    __syncthreads();
    for (int i = r0; i < n8; i += rstep) Mdst[i * n8 + c0] = T5[i * ld + c0];
    // M is what the other CTAs wait for: arrive now, finish the top rows, then wait
    grid_barrier_arrive(&a.bar[0], epoch);
    arrived = true;
    // top rows: R = S R~ in the panel rows (zeros below the diagonal)
    for (int e = tid; e < n * n; e += kFT) {
      const int l = e / n, i = e - l * n;
      if (i < a.rrows) a.Rdst[i + (int64_t)l * a.ldr] = i <= l ? s_sign[i] * Rt[i * ld + l] : 0.0;
    }
    for (int j = tid; j < n; j += kFT) a.tau[j] = fabs(s_c[j]) + 1.0;
    if (tid == 0) {
      if (a.msu != nullptr) a.st->degenerate = s_degen;
      // _panel_rank: every column usable; level-2 counters of the
      // column-by-column reflections this path replaces
      int64_t l2 = a.l2_extra;
      for (int j = 0; j + 1 < n; ++j) l2 += (a.mm - j) * (int64_t)(n - j - 1);
      a.st->usable = a.usable_total > 0 ? a.usable_total : n;
      a.st->level2 += 4 * l2;
      a.st->l2bytes += 16 * l2;
    }
    sub(8);
  } else if (me == 1 && a.msu != nullptr) {
    // sample update's M = S11 R11^{-1} (randomized.py:107-135): R11 = S R~,
    // R~^{-1} = R1^{-1} (I - F) to O(|F|^2), so M = S11 R1^{-1} (I - F) S.
    // A committed panel cleared the degenerate guard (same threshold).
    // (W0 may hold this CTA's resident panel rows; W2 = R1^{-1} since phase B)
    for (int i = r0; i < n8; i += rstep) {
      const int l = c0, e = i * n8 + l;
      double f = 0.0;
      if (i <= l && l < n) {
        const double E = ldcg(a.gmat + 3 * nn + e) - (i == l ? 1.0 : 0.0);
        f = (i == l) ? 0.5 * E : E;
      }
      W3[i * ld + l] = f;
      W4[i * ld + l] = (i < n && l < n) ? a.S11[i + (int64_t)l * a.lds11] : 0.0;
    }
    for (int j = tid; j < n8; j += kFT) s_sign[j] = ldcg(gxs + j);
    __syncthreads();
    chunk_mm<false, true>(W4, W2, W5, n8, n8, ld);   // S11 R1^{-1}
    __syncthreads();
    chunk_mm<false, true>(W5, W3, W4, n8, n8, ld);   // (S11 R1^{-1}) F
    __syncthreads();
    for (int e = tid; e < n * n; e += kFT) {
      const int l = e / n, i = e - l * n;
      a.msu[i + (int64_t)l * n] = s_sign[l] * (W5[i * ld + l] - W4[i * ld + l]);
    }
  } else if (me == 2 && a.T != nullptr) {
    // compact-WY T of the reconstructed reflectors: U = -T Y1^T, so
    // T = -U Y1^{-T} (kernels.py:139-147 builds the same T by recurrence)
    for (int i = r0; i < n8; i += rstep) {
      W1[i * ld + c0] = ldcg(gxU + i * n8 + c0);
      W3[i * ld + c0] = i == c0 ? 1.0 : (i < c0 ? ldcg(gxL + c0 * n8 + i) : 0.0);   // Y1^T
    }
    for (int j = tid; j < n8; j += kFT) {
      s_dinv[j] = 1.0;
      s_sign[j] = ldcg(gxs + j);
    }
    __syncthreads();
    upper_inverse<kFT>(W3, s_dinv, W4, W5, n8, ld);   // X = Y1^{-T}
    __syncthreads();
    chunk_mm<true, true>(W1, W4, W5, n8, n8, ld);     // U X = -T
    __syncthreads();
    for (int e = tid; e < n * n; e += kFT) {
      const int l = e / n, i = e - l * n;
      a.T[i + (int64_t)l * a.ldt] = i <= l ? -W5[i * ld + l] : 0.0;
    }
    if (a.a12 != nullptr) {
      // X = T^T G with G = Y1^T C_top + M^T H  =>  X = A1^T C_top + A2^T H,
      // A1 = Y1 T, A2 = M T = -R1^{-1} (I - F) S Y1^{-T} (U^{-1} U cancels, so
      // A2 does not wait for CTA 0's M); block_finish_kernel applies them
      for (int i = r0; i < n8; i += rstep)   // Y1 (unit lower)
        W3[i * ld + c0] = i == c0 ? 1.0 : (i > c0 ? ldcg(gxL + i * n8 + c0) : 0.0);
      __syncthreads();
      chunk_mm<false, true>(W3, W5, W1, n8, n8, ld);   // Y1 (-T)
      __syncthreads();
      for (int e = tid; e < n * n; e += kFT) {   // row-major: block_finish's staging layout
        const int i = e / n, l = e - i * n;
        a.a12[e] = -W1[i * ld + l];
      }
      __syncthreads();
      for (int i = r0; i < n8; i += rstep) {
        const int l = c0, e = i * n8 + l;
        double f = 0.0;
        if (i <= l && l < n) {
          const double E = ldcg(a.gmat + 3 * nn + e) - (i == l ? 1.0 : 0.0);
          f = (i == l) ? 0.5 * E : E;
        }
        W1[i * ld + l] = f;                              // F
        W3[i * ld + l] = s_sign[i] * W4[i * ld + l];     // N = S Y1^{-T}
      }
      __syncthreads();
      chunk_mm<true, true>(W1, W3, W5, n8, n8, ld);      // F N
      __syncthreads();
      for (int i = r0; i < n8; i += rstep) W3[i * ld + c0] -= W5[i * ld + c0];   // (I - F) N
      __syncthreads();
      chunk_mm<true, true>(W2, W3, W1, n8, n8, ld);      // R1^{-1} (I - F) N = -A2
      __syncthreads();
      for (int e = tid; e < n * n; e += kFT) {
        const int i = e / n, l = e - i * n;
        a.a12[(int64_t)n * n + e] = -W1[i * ld + l];
      }
    }
  }
  mark(6);
  if (!arrived) grid_barrier_arrive(&a.bar[0], epoch);
  grid_barrier_wait(&a.bar[0], epoch);

  // ---- phase C: Y_below = P_below M, zeros below the diagonal of the panel rows
  for (int i = r0; i < n8; i += rstep) W2[i * ld + c0] = ldcg(Mdst + i * n8 + c0);
  if (!resident && me < a.nchunks) load_regs(a, me, pre);
  for (int64_t ch = me; ch < a.nchunks; ch += Q) {
    __syncthreads();
    if (!resident) store_regs(a, pre, W0);
    __syncthreads();
    if (!resident && ch + Q < a.nchunks) load_regs(a, ch + Q, pre);
    chunk_mm<false, true>(W0, W2, W1, kFRows, n8, ld);
    __syncthreads();
    const int64_t g0 = ch * kFRows;
    for (int e = tid; e < kFRows * n; e += kFT) {
      const int c = e >> 6, r = e & (kFRows - 1);
      const int64_t gr = g0 + r;
      if (gr < n || gr >= a.mm) continue;
      a.Y[gr + (int64_t)c * a.ldy] = W1[r * ld + c];
      if (gr < a.rrows && !a.defer_zero) a.Rdst[gr + (int64_t)c * a.ldr] = 0.0;
    }
  }
  mark(7);
  finish();
}

}  // namespace

bool panel_fast_eligible(const Handle& h, int64_t mm, int64_t bw) {
  if (!h.fast_panel || bw < 2 || bw > kFMaxBw || mm < 2 * bw) return false;
  // the kernel's layouts (log2 strides, the recursive block inverse) need a
  // power-of-two padded width: n8 in {8, 16, 32, 64}
  const int n8 = (int)((bw + 7) / 8 * 8);
  return n8 == 8 || n8 == 16 || n8 == 32 || n8 == 64;
}

const int* panel_fast(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
                      const PanelOut& out, double tol, Status* st, cudaStream_t s,
                      bool abort_on_decline, int64_t i0, int max_ctas, bool defer_zero,
                      const double** m_rowmajor, int64_t* m_ld, const double* S11,
                      int64_t lds11, double* msu, double* a12, int64_t l2_extra,
                      int usable_total, bool degen_commit) {
  if (!panel_fast_eligible(h, mm, bw)) return nullptr;
  const int n8 = (int)((bw + 7) / 8 * 8);
  const int ld = n8 + h.fast_panel_pad;
  const int64_t nchunks = (mm + kFRows - 1) / kFRows;
  int Q = (int)std::min<int64_t>(h.num_sms, nchunks);
  if (h.fast_panel_max_ctas > 0) Q = std::min(Q, h.fast_panel_max_ctas);
  if (max_ctas > 0) Q = std::min(Q, max_ctas);
  Q = std::max(Q, 3);   // CTAs 1 and 2 carry the second serial section's side products
  const size_t smem = (size_t)6 * kFRows * ld * 8;
  const int nn = n8 * n8;
  FastArgs a{};
  a.mm = mm; a.n = (int)bw; a.n8 = n8; a.ld = ld;
  a.P = P; a.ldp = ldp;
  a.Rdst = out.Rdst; a.ldr = out.ldr; a.rrows = out.rrows;
  a.Y = out.Y; a.ldy = out.ldy; a.tau = out.tau;
  a.T = out.T; a.ldt = out.ldt;
  a.tol = tol;
  a.guard = tol >= 0.0 ? tol * (kEps34 / kEps) : -1.0;
  a.nchunks = nchunks;
  a.st = st;
  a.abort_on_decline = abort_on_decline ? 1 : 0;
  a.defer_zero = defer_zero ? 1 : 0;
  a.S11 = S11; a.lds11 = lds11; a.msu = S11 != nullptr ? msu : nullptr;
  a.a12 = out.T != nullptr ? a12 : nullptr;
  a.l2_extra = l2_extra;
  a.usable_total = usable_total;
  a.degen_commit = (degen_commit && S11 != nullptr) ? 1 : 0;
  a.i0 = i0;
  a.bar = (unsigned int*)h.buf("pf_bar", 64, s);
  static void* zeroed = nullptr;
  if (zeroed != (void*)a.bar) {
    RQ_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
    zeroed = a.bar;
  }
  a.gpart = (double*)h.buf("pf_part", (size_t)Q * nn * 8, s);
  a.gmat = (double*)h.buf("pf_mat", (size_t)5 * nn * 8, s);
  a.gx = (double*)h.buf("pf_x", ((size_t)2 * nn + n8) * 8, s);
  // on commit, M = R1^{-1} (I - F) S U^{-1} (Y_below = P_below M) is left
  // row-major in gmat[4]: as a column-major matrix with ld n8 it is M^T
  if (m_rowmajor != nullptr) *m_rowmajor = a.gmat + 4 * nn;
  if (m_ld != nullptr) *m_ld = n8;
  a.dbg = h.dbg;
  kernel_attr((const void*)panel_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)std::max<size_t>(smem, 48 * 1024));
  {
    ProfScope prof(h, kProfPanel, 6.0 * mm * bw * bw, 24.0 * mm * bw, s);
    void* args[] = {&a};
    RQ_CUDA(cudaLaunchCooperativeKernel((void*)panel_fast_kernel, dim3(Q), dim3(kFT), args, smem,
                                        s));
    RQ_CHECK_LAUNCH();
    count_launch();
  }
  return (const int*)&a.bar[4];
}

}  // namespace rq
