// Small / memory-bound kernels of the block loop: sample update (K3),
// swap replay (K6), Frobenius norm (K10), copies, permutation scatter and
// the standalone T factor.
#include "runtime.hpp"
#include "tri.cuh"

namespace rq {

namespace {

// ---------------------------------------------------------------- K3
// B_new[:, c] = [S12[:, c] - S11 R11^{-1} R12[:, c];  S22[:, c]]
// (randomized.py:107-135).  One thread per sample column; R11 staged in
// shared memory, the solve vector kept column-per-thread in shared memory.
constexpr int kSuThreads = 64;

__global__ void __launch_bounds__(kSuThreads) sample_update_kernel(
    int ell, int b, int64_t n2, const double* __restrict__ S, int64_t lds,
    const double* __restrict__ R11, const double* __restrict__ R12, int64_t ldr, double thresh,
    double* __restrict__ Bn, int64_t ldb, Status* st, int abort_on_degenerate, int64_t i0,
    int r11_staged) {
  if (aborted(st)) return;
  extern __shared__ __align__(16) double sm[];
  // R11 staged in shared memory (b x b, col-major ld b) while it fits beside
  // the solve vectors; wider blocks (b > ~140) read it through L1/L2
  const double* r11 = r11_staged ? sm : R11;
  const int64_t ld11 = r11_staged ? b : ldr;
  double* xs = sm + (r11_staged ? (size_t)b * b : 0);     // b x kSuThreads
  const int tid = threadIdx.x;
  // degenerate test first, as the reference raises before solving (:117)
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int j = tid; j < b; j += kSuThreads)
    if (fabs(R11[j + (size_t)j * ldr]) < thresh) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (blockIdx.x == 0 && tid == 0) {
      st->degenerate = 1;
      if (abort_on_degenerate) {
        st->abort_i0 = i0;
        __threadfence();
        st->abort = kAbortDegenerate;
      }
    }
    return;
  }
  if (blockIdx.x == 0 && tid == 0) st->degenerate = 0;
  if (r11_staged) {
    for (int e = tid; e < b * b; e += kSuThreads) {
      const int i = e % b, j = e / b;
      sm[e] = R11[i + (size_t)j * ldr];
    }
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * kSuThreads + tid;
  if (c >= n2) return;
  double* x = xs + tid;
  for (int i = 0; i < b; ++i) x[i * kSuThreads] = R12[i + (size_t)c * ldr];
  // back substitution (np.linalg.solve on the upper-triangular R11)
  for (int i = b - 1; i >= 0; --i) {
    const double xi = __ddiv_rn(x[i * kSuThreads], r11[i + i * ld11]);
    x[i * kSuThreads] = xi;
    for (int l = 0; l < i; ++l)
      x[l * kSuThreads] = __fma_rn(-r11[l + i * ld11], xi, x[l * kSuThreads]);
  }
  // B1 = S12 - S11 @ X   (S11 upper triangular: only l >= i contribute)
  const double* s12 = S + (size_t)(b + c) * lds;
  double* out = Bn + (size_t)c * ldb;
  for (int i = 0; i < b; ++i) {
    double acc = 0.0;
    for (int l = i; l < b; ++l) acc = __fma_rn(__ldg(S + i + (size_t)l * lds), x[l * kSuThreads], acc);
    out[i] = __dsub_rn(s12[i], acc);
  }
  for (int i = b; i < ell; ++i) out[i] = s12[i];
}

// Register-resident variant for b in {16, 32, 64}: thread per column, the
// solve vector lives in registers, R11 and S11 are staged in shared memory
// (broadcast reads).  X = R11^{-1} R12 by back substitution with the
// reciprocal diagonal (OpenBLAS dtrsm, behind np.linalg.solve, also scales by
// the inverted diagonal), then B1 = S12 - S11 X.
template <int B>
__global__ void __launch_bounds__(128) sample_update_reg_kernel(
    int ell, int64_t n2, const double* __restrict__ S, int64_t lds,
    const double* __restrict__ R11, const double* __restrict__ R12, int64_t ldr, double thresh,
    double* __restrict__ Bn, int64_t ldb, Status* st, int abort_on_degenerate, int64_t i0) {
  if (aborted(st)) return;
  extern __shared__ __align__(16) double dyn[];
  double* r11 = dyn;              // r11[l + i*B] = R11[l, i]
  double* s11 = dyn + B * B;      // s11[i + l*B] = S11[i, l]
  double* rinv = dyn + 2 * B * B;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int j = tid; j < B; j += blockDim.x) {
    const double d = R11[j + (size_t)j * ldr];
    if (fabs(d) < thresh) s_bad = 1;
    rinv[j] = 1.0 / d;
  }
  for (int e = tid; e < B * B; e += blockDim.x) {
    const int i = e % B, l = e / B;
    r11[e] = R11[i + (size_t)l * ldr];
    s11[e] = S[i + (size_t)l * lds];
  }
  __syncthreads();
  if (s_bad) {
    if (blockIdx.x == 0 && tid == 0) {
      st->degenerate = 1;
      if (abort_on_degenerate) {
        st->abort_i0 = i0;
        __threadfence();
        st->abort = kAbortDegenerate;
      }
    }
    return;
  }
  if (blockIdx.x == 0 && tid == 0) st->degenerate = 0;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + tid;
  if (c >= n2) return;
  double x[B];
  const double* rc = R12 + (size_t)c * ldr;
#pragma unroll
  for (int i = 0; i < B; ++i) x[i] = rc[i];
#pragma unroll
  for (int i = B - 1; i >= 0; --i) {
    x[i] = __dmul_rn(x[i], rinv[i]);
#pragma unroll
    for (int l = 0; l < i; ++l) x[l] = __fma_rn(-r11[l + i * B], x[i], x[l]);
  }
  const double* s12 = S + (size_t)(B + c) * lds;
  double* out = Bn + (size_t)c * ldb;
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int l = i; l < B; ++l) acc = __fma_rn(s11[i + l * B], x[l], acc);
    out[i] = __dsub_rn(s12[i], acc);
  }
  for (int i = B; i < ell; ++i) out[i] = s12[i];
}

// Sample update as a GEMM (randomized.py:107-135): top = S12 - S11 R11^{-1}
// R12 = S12 - M R12 with M = S11 R11^{-1} (b x b).  One CTA checks the
// degenerate guard (|R11_jj| < eps^3/4 ||A||_F, randomized.py:117) and forms M
// (recursive DMMA triangular inverse, tri.cuh); the rank-b update kernel then
// applies M to R12.  The per-column back substitution it replaces was a
// latency chain (66 us at n2 = 8128).  M is written column-major (ld b).
template <int B>
__global__ void __launch_bounds__(256) su_prep_kernel(const double* __restrict__ S, int64_t lds,
                                                      const double* __restrict__ R11, int64_t ldr,
                                                      double thresh, double* __restrict__ M,
                                                      Status* st, int abort_on_degenerate,
                                                      int64_t i0) {
  if (aborted(st)) return;
  constexpr int LD = B + 1;
  extern __shared__ __align__(16) double su_sm[];
  double* U = su_sm;
  double* X = U + B * LD;
  double* Tm = X + B * LD;
  double* S11 = Tm + B * LD;
  double* dinv = S11 + B * LD;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int e = tid; e < B * B; e += blockDim.x) {
    const int i = e % B, l = e / B;   // column-major reads
    U[i * LD + l] = i <= l ? R11[i + (size_t)l * ldr] : 0.0;
    S11[i * LD + l] = S[i + (size_t)l * lds];
  }
  for (int j = tid; j < B; j += blockDim.x) {
    const double d = R11[j + (size_t)j * ldr];
    if (fabs(d) < thresh) s_bad = 1;
    dinv[j] = 1.0 / d;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      st->degenerate = 1;
      if (abort_on_degenerate) {
        st->abort_i0 = i0;
        __threadfence();
        st->abort = kAbortDegenerate;
      }
    }
    return;
  }
  if (tid == 0) st->degenerate = 0;
  upper_inverse<256>(U, dinv, X, Tm, B, LD);
  __syncthreads();
  // M = S11 X (X upper): one 8x8 tile per warp iteration
  const int warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fk = lane & 3;
  constexpr int nt = B / 8;
  for (int t = warp; t < nt * nt; t += 8) {
    const int ti = t / nt, tj = t % nt;
    double acc[2] = {0.0, 0.0};
    tile_mm(S11 + ti * 8 * LD, X + tj * 8, 8 * (tj + 1), LD, acc);
    const int r = ti * 8 + fr, c = tj * 8 + 2 * fk;
    M[r + (size_t)c * B] = acc[0];
    M[r + (size_t)(c + 1) * B] = acc[1];
  }
}

// One-launch replay of the select swaps (randomized.py:138-147): the net
// permutation of the <= 2 got touched positions is planned redundantly by
// every block (<= 256 pivots, one backward trace per position), then each block moves ITS rows of every moved
// column through shared memory -- all sources of a row chunk are read before
// any destination is written, and blocks own disjoint rows, so no scratch
// buffer or second pass is needed.  Units: row chunks of the work matrix, of
// R's columns and of W's rows (TRQRCP followers).  Block 0 also permutes
// Permutation.forward and appends the swap log.
constexpr int kSwapRows = 32;
__global__ void __launch_bounds__(256) swap_fused_kernel(const int64_t* __restrict__ piv, int64_t i0,
                                                          SwapTargets t, Status* st, int units_w,
                                                          int units_r) {
  if (aborted(st)) return;
  const int got = (int)st->got;
  extern __shared__ double sbuf[];                 // [2 got][kSwapRows]
  __shared__ int pv[256], lsrc[512], ldst[512];
  __shared__ int s_nlive;
  __shared__ int64_t s_nswaps;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_nlive = 0;
    s_nswaps = st->nswaps;
  }
  for (int e = tid; e < got; e += blockDim.x) pv[e] = (int)piv[e];
  __syncthreads();
  // touched positions: q < got, and each pivot position q >= got once (its
  // first occurrence).  Position q's final content comes from the position
  // found by replaying the transpositions (k, piv[k]) backwards -- one
  // independent trace per thread instead of a serial replay.
  for (int e = tid; e < 2 * got; e += blockDim.x) {
    int q;
    bool cand = true;
    if (e < got) {
      q = e;
    } else {
      const int k0 = e - got;
      q = pv[k0];
      cand = q >= got;
      for (int kk = 0; kk < k0 && cand; ++kk) cand = pv[kk] != q;
    }
    if (!cand) continue;
    int sp = q;
    for (int k = got - 1; k >= 0; --k) {
      const int pk = pv[k];
      sp = sp == k ? pk : (sp == pk ? k : sp);
    }
    if (sp != q) {
      const int i = atomicAdd(&s_nlive, 1);
      lsrc[i] = sp;
      ldst[i] = q;
    }
  }
  __syncthreads();
  const int nl = s_nlive;
  if (blockIdx.x == 0) {
    int64_t* pbuf = (int64_t*)sbuf;
    for (int i = tid; i < nl; i += blockDim.x) pbuf[i] = t.perm[i0 + lsrc[i]];
    for (int e = tid; e < got; e += blockDim.x)
      if (s_nswaps + e < t.log_cap) {   // swap log: stores only
        t.log[2 * (s_nswaps + e)] = i0 + e;
        t.log[2 * (s_nswaps + e) + 1] = i0 + pv[e];
      }
    __syncthreads();
    for (int i = tid; i < nl; i += blockDim.x) t.perm[i0 + ldst[i]] = pbuf[i];
    if (tid == 0) st->nswaps = s_nswaps + got;
    __syncthreads();
  }
  if (nl == 0) return;
  // my unit: a chunk of kSwapRows "rows" of one follower array
  int u = blockIdx.x;
  double* base;
  int64_t rows, rstride, cstride;
  if (u < units_w) {
    base = t.work; rows = t.m; rstride = 1; cstride = t.ldw;
  } else if ((u -= units_w) < units_r) {
    base = t.Rf; rows = t.rf_rows; rstride = 1; cstride = t.ldrf;
  } else {
    u -= units_r;
    base = t.Wf; rows = t.wf_cols; rstride = t.ldwf; cstride = 1;
  }
  const int64_t r0 = (int64_t)u * kSwapRows;
  const int nr = (int)imin64(kSwapRows, rows - r0);
  // eight independent loads in flight per thread (one dependent round trip
  // per element made this phase latency bound)
  const int tot = nl * kSwapRows;
  for (int e0 = tid; e0 < tot; e0 += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      const int i = e / kSwapRows, r = e - i * kSwapRows;
      v[u] = (e < tot && r < nr) ? base[(r0 + r) * rstride + (i0 + lsrc[i]) * cstride] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < tot) sbuf[e] = v[u];
    }
  }
  __syncthreads();
  for (int e = tid; e < nl * kSwapRows; e += blockDim.x) {
    const int i = e / kSwapRows, r = e - i * kSwapRows;
    if (r < nr) base[(r0 + r) * rstride + (i0 + ldst[i]) * cstride] = sbuf[e];
  }
}

// ---------------------------------------------------------------- K10
constexpr int kNormBlocks = 296, kNormThreads = 256;
__global__ void sumsq_partial_kernel(const double* A, int64_t m, int64_t n, int64_t lda,
                                     double* part) {
  __shared__ double red[kNormThreads];
  double acc = 0.0;
  const int64_t total = m * n;
  for (int64_t e = (int64_t)blockIdx.x * kNormThreads + threadIdx.x; e < total;
       e += (int64_t)kNormBlocks * kNormThreads) {
    const double v = A[(e % m) + (e / m) * lda];
    acc = __fma_rn(v, v, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kNormThreads / 2; s; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void sumsq_final_kernel(const double* part, double* out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < kNormBlocks; ++b) t = __dadd_rn(t, part[b]);
    *out = sqrt(t);
  }
}

__global__ void copy2d_kernel(const double* src, int64_t lds, double* dst, int64_t ldd,
                              int64_t rows, int64_t cols, const Status* st) {
  if (aborted(st)) return;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    dst[r + c * ldd] = src[r + c * lds];
  }
}
// Two-half panel guard (driver.cu panel_halves).  The reference eliminates a
// panel on a copy and commits it only once its whole R diagonal is confirmed
// (randomized.py:221-239); the two-half panel writes its first half in place
// before the second half is factored.  restore = 0: snapshot the selected
// columns and the level-2 counters (skipped when the queue already aborted).
// restore = 1: if the block's fast panel declined (Status.abort ==
// kAbortPanelFast at i0), put the columns and counters back and clear the
// first half's reflectors, so the rewind redoes the panel on the original
// columns exactly as the reference would.
__global__ void halves_guard_kernel(double* work, int64_t ldw, int64_t mm, int64_t cols,
                                    double* snap, int64_t* sst, Status* st, int restore,
                                    int64_t i0, double* Y, int64_t ldy, double* tau) {
  if (!restore) {
    if (aborted(st)) return;
  } else {
    const int code = *((volatile const int*)&st->abort);
    if (code != kAbortPanelFast || st->abort_i0 != i0) return;
  }
  const int64_t total = mm * cols;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t e = t0; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % mm, c = e / mm;
    if (!restore) {
      snap[e] = work[r + c * ldw];
    } else {
      work[r + c * ldw] = snap[e];
      Y[r + c * ldy] = 0.0;
    }
  }
  if (t0 == 0) {
    if (!restore) {
      sst[0] = st->level2;
      sst[1] = st->l2bytes;
    } else {
      st->level2 = sst[0];
      st->l2bytes = sst[1];
    }
  }
  if (restore && t0 < cols) tau[t0] = 0.0;
}
// NormTracker.downdate / downdate_norms (kernels.py:189-192, 225-233):
// new_sq = max(norm^2 - row^2, 0), in numpy's operation order (bit-identical);
// with orig_sq, unsafe[j] = new_sq < guard * orig_sq[j] (the caller recomputes
// those columns exactly).
__global__ void norm_downdate_kernel(const double* norms, const double* row, int64_t inc,
                                     int64_t n, const double* orig_sq, double guard, double* out,
                                     int32_t* unsafe) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double v = norms[j], r = row[j * inc];
    const double sq = fmax(__dsub_rn(__dmul_rn(v, v), __dmul_rn(r, r)), 0.0);
    out[j] = sqrt(sq);
    if (unsafe != nullptr) unsafe[j] = orig_sq != nullptr && sq < __dmul_rn(guard, orig_sq[j]);
  }
}
__global__ void fill2d_kernel(double* dst, int64_t ldd, int64_t rows, int64_t cols, double v,
                              const Status* st) {
  if (aborted(st)) return;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[(e % rows) + (e / rows) * ldd] = v;
}
__global__ void identity_kernel(double* dst, int64_t ldd, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    dst[r + c * ldd] = r == c ? 1.0 : 0.0;
  }
}
// 32x32 tiled transpose: dst (cols x rows) = src (rows x cols)^T
__global__ void transpose_kernel(const double* src, int64_t lds, double* dst, int64_t ldd,
                                 int64_t rows, int64_t cols) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[r + c * lds];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + k;
    if (r < rows && c < cols) dst[c + r * ldd] = tile[threadIdx.x][k];
  }
}
// dst[:, perm[i]] = src[:, i]  (Permutation.restore, kernels.py:107-111)
__global__ void scatter_cols_kernel(const double* src, int64_t lds, const int64_t* perm,
                                    double* dst, int64_t ldd, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % rows, c = e / rows;
    dst[r + perm[c] * ldd] = src[r + c * lds];
  }
}
// T recurrence from the Gram matrix G (nb x nb, upper part used):
// T[:j, j] = -tau_j * (T[:j, :j] @ G[:j, j]), T[j, j] = tau_j (kernels.py:139-147).
// T lives in shared memory while it is built (nb <= 128), else in place.
__global__ void t_recurrence_kernel(const double* __restrict__ G, int64_t ldg,
                                    const double* __restrict__ tau, int nb, double* T,
                                    int64_t ldt, const Status* st) {
  if (aborted(st)) return;
  extern __shared__ double tsm[];
  const bool in_smem = nb <= 128;
  double* Tw = in_smem ? tsm : T;
  const int64_t ldw = in_smem ? nb : ldt;
  double* tmp = in_smem ? tsm + (size_t)nb * nb : tsm;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Tw[(e % nb) + (e / nb) * ldw] = 0.0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double tj = tau[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
      double t = 0.0;
      for (int l = i; l < j; ++l) t = __fma_rn(Tw[i + (size_t)l * ldw], G[l + (size_t)j * ldg], t);
      tmp[i] = t;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < j; i += blockDim.x) Tw[i + (size_t)j * ldw] = __dmul_rn(-tj, tmp[i]);
    if (threadIdx.x == 0) Tw[j + (size_t)j * ldw] = tj;
    __syncthreads();
  }
  if (in_smem)
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x)
      T[(e % nb) + (size_t)(e / nb) * ldt] = Tw[e];
}

// The same T as the recurrence above, as the inverse of U = striu(Y^T Y) +
// diag(1/tau): the recurrence is exactly column-wise back substitution for
// U^{-1} (T[:j, j] = -T[:j, :j] U[:j, j] / U[j, j], U[j, j] = 1/tau_j), so any
// triangular inversion gives T; this one is the recursive DMMA block inverse
// of tri.cuh (dinv = tau, no divisions).  A tau_j = 0 reflector is the
// identity: its row and column of T are zero (the recurrence's result), so
// index j is decoupled (unit diagonal, zero off-diagonals) and zeroed after.
__global__ void __launch_bounds__(256, 1) t_inverse_kernel(const double* __restrict__ G, int64_t ldg,
                                                           const double* __restrict__ tau, int nb,
                                                           double* T, int64_t ldt,
                                                           const Status* st) {
  if (aborted(st)) return;
  constexpr int kLd = 65;
  extern __shared__ __align__(16) double tsm_inv[];
  double* U = tsm_inv;
  double* X = U + 64 * kLd;
  double* Tmp = X + 64 * kLd;
  __shared__ double dinv[64];
  // upper_inverse joins pairs of blocks level by level: a power-of-2 size
  const int n8 = nb <= 8 ? 8 : (nb <= 16 ? 16 : (nb <= 32 ? 32 : 64));
  for (int e = threadIdx.x; e < n8 * n8; e += 256) {
    const int i = e / n8, l = e - i * n8;
    double u = 0.0;
    if (i < l && l < nb && tau[i] != 0.0 && tau[l] != 0.0) u = G[i + (int64_t)l * ldg];
    U[i * kLd + l] = u;
  }
  for (int j = threadIdx.x; j < n8; j += 256) dinv[j] = (j < nb && tau[j] != 0.0) ? tau[j] : 1.0;
  __syncthreads();
  upper_inverse<256>(U, dinv, X, Tmp, n8, kLd);
  __syncthreads();
  for (int e = threadIdx.x; e < nb * nb; e += 256) {
    const int i = e % nb, l = e / nb;
    double t = i <= l ? X[i * kLd + l] : 0.0;
    if (i == l && tau[i] == 0.0) t = 0.0;
    T[i + (int64_t)l * ldt] = t;
  }
}

// b = 128 (cfg5) sample update prep: the degenerate verdict exactly as
// su_prep_kernel, then the inverses of the two diagonal 64-blocks of R11 =
// [[A, B], [0, C]] (recursive DMMA inverse, tri.cuh) into Ainv / Cinv
// (column-major, ld 64); the caller assembles R11^{-1} and M = S11 R11^{-1}
// with GEMMs.
__global__ void __launch_bounds__(256, 1) su_prep_wide_kernel(const double* __restrict__ R11,
                                                              int64_t ldr, int b, double thresh,
                                                              double* Ainv, double* Cinv,
                                                              int64_t ldi, Status* st,
                                                              int abort_on_degenerate,
                                                              int64_t i0) {
  if (aborted(st)) return;
  constexpr int LD = 65;
  extern __shared__ __align__(16) double wsm[];
  double* U = wsm;
  double* X = U + 64 * LD;
  double* Tm = X + 64 * LD;
  __shared__ double dinv[64];
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int j = tid; j < b; j += blockDim.x)
    if (fabs(R11[j + (size_t)j * ldr]) < thresh) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      st->degenerate = 1;
      if (abort_on_degenerate) {
        st->abort_i0 = i0;
        __threadfence();
        st->abort = kAbortDegenerate;
      }
    }
    return;
  }
  if (tid == 0) st->degenerate = 0;
  for (int half = 0; half < 2; ++half) {
    const int o = 64 * half;
    for (int e = tid; e < 64 * 64; e += blockDim.x) {
      const int i = e % 64, l = e / 64;
      U[i * LD + l] = i <= l ? R11[(o + i) + (size_t)(o + l) * ldr] : 0.0;
    }
    for (int j = tid; j < 64; j += blockDim.x) dinv[j] = 1.0 / R11[(o + j) + (size_t)(o + j) * ldr];
    __syncthreads();
    upper_inverse<256>(U, dinv, X, Tm, 64, LD);
    __syncthreads();
    double* dst = half ? Cinv : Ainv;
    for (int e = tid; e < 64 * 64; e += blockDim.x) {
      const int i = e % 64, l = e / 64;
      dst[i + (size_t)l * ldi] = i <= l ? X[i * LD + l] : 0.0;
    }
    __syncthreads();
  }
}

// column_norms (kernels.py:184-186) = np.linalg.norm(A, axis=0), bit for bit:
// numpy sums the rounded squares pairwise along a contiguous (F-order) column
// and strictly in row order across a C-order array (axis 0 is then the outer
// loop), so the caller names the layout it mirrors.
__global__ void col_norms_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                 int sequential, double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double* x = A + j * lda;
  double s;
  if (sequential) {
    s = 0.0;
    for (int64_t i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(x[i], x[i]));
  } else {
    s = pairwise_sumsq(x, (int)m, 1);
  }
  out[j] = sqrt(s);
}

int grid_for(int64_t total, int num_sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 16LL * num_sms));
}

}  // namespace

void sample_update_pre(Handle& h, int64_t ell, int64_t b, int64_t n2, const double* S,
                       int64_t lds, const double* M, const double* R12, int64_t ldr,
                       double* Bnew, int64_t ldb, Status* st, cudaStream_t s) {
  if (n2 <= 0) return;
  ProfScope prof(h, kProfSampleUpd, 3.0 * b * b * n2, 8.0 * (2 * ell * n2 + b * b), s);
  // one launch: Bnew[:b] = S12 - M R12 and Bnew[b:] = S22 (rank-b kernel with a
  // separate C source and pass-through rows); else copy + GEMM
  if (rank_update(h, b, n2, b, M, b, R12, ldr, Bnew, ldb, s, st, kProfSampleUpd, 0, nullptr,
                  S + (size_t)b * lds, lds, (int)(ell - b)))
    return;
  copy2d(S + (size_t)b * lds, lds, Bnew, ldb, ell, n2, s, st);
  if (!rank_update(h, b, n2, b, M, b, R12, ldr, Bnew, ldb, s, st, kProfSampleUpd))
    gemm(h, false, false, b, n2, b, -1.0, M, b, R12, ldr, 1.0, Bnew, ldb, s, st, kProfSampleUpd);
}

void sample_update(Handle& h, int64_t ell, int64_t b, int64_t n2, const double* S, int64_t lds,
                   const double* R11, const double* R12, int64_t ldr, double frob,
                   double* Bnew, int64_t ldb, Status* st, bool abort_on_degenerate, int64_t i0,
                   cudaStream_t s) {
  if (h.su_gemm && (b == 16 || b == 32 || b == 64)) {
    ProfScope prof(h, kProfSampleUpd, 3.0 * b * b * n2, 8.0 * (2 * ell * n2 + b * b), s);
    double* M = (double*)h.buf("su_M", (size_t)b * b * 8, s);
    const double th = kEps34 * frob;
    const int ab = abort_on_degenerate ? 1 : 0;
    const size_t psm = ((size_t)4 * b * (b + 1) + b) * 8;
    kernel_attr((const void*)su_prep_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)(((size_t)4 * 64 * 65 + 64) * 8));
    if (b == 16) su_prep_kernel<16><<<1, 256, psm, s>>>(S, lds, R11, ldr, th, M, st, ab, i0);
    else if (b == 32) su_prep_kernel<32><<<1, 256, psm, s>>>(S, lds, R11, ldr, th, M, st, ab, i0);
    else su_prep_kernel<64><<<1, 256, psm, s>>>(S, lds, R11, ldr, th, M, st, ab, i0);
    RQ_CHECK_LAUNCH();
    count_launch();
    if (n2 > 0) {
      // B_new = S[:, b:] with its top b rows then reduced by M R12; the
      // degenerate verdict (non-speculative caller) leaves B_new unused
      const Status* pred = abort_on_degenerate ? st : nullptr;
      copy2d(S + (size_t)b * lds, lds, Bnew, ldb, ell, n2, s, pred);
      if (!rank_update(h, b, n2, b, M, b, R12, ldr, Bnew, ldb, s, pred, kProfSampleUpd))
        gemm(h, false, false, b, n2, b, -1.0, M, b, R12, ldr, 1.0, Bnew, ldb, s, pred,
             kProfSampleUpd);
    }
    return;
  }
  if (h.su_gemm && b == 128) {
    // R11^{-1} = [[A^-1, -A^-1 B C^-1], [0, C^-1]], M = S11 R11^{-1}, then
    // B_new[:b] = S12 - M R12 as in the b <= 64 path
    ProfScope prof(h, kProfSampleUpd, 3.0 * b * b * n2, 8.0 * (2 * ell * n2 + b * b), s);
    double* Ri = (double*)h.buf("su_R11inv", (size_t)128 * 128 * 8, s);
    double* W = (double*)h.buf("su_wide_tmp", (size_t)64 * 64 * 8, s);
    double* M = (double*)h.buf("su_M", (size_t)128 * 128 * 8, s);
    const int ab = abort_on_degenerate ? 1 : 0;
    constexpr size_t wsm = (size_t)3 * 64 * 65 * 8;
    kernel_attr((const void*)su_prep_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)wsm);
    double* Ri22 = Ri + 64 + (size_t)64 * 128;
    fill2d(Ri + 64, 128, 64, 64, 0.0, s, st);   // the zero block below A^-1
    su_prep_wide_kernel<<<1, 256, wsm, s>>>(R11, ldr, 128, kEps34 * frob, Ri, Ri22, 128, st, ab,
                                            i0);
    RQ_CHECK_LAUNCH();
    count_launch();
    // the Status predicate skips the rest after a degenerate verdict (the
    // non-speculative caller reads Status.degenerate and discards B_new)
    const Status* pred = st;
    // X12 = -A^-1 (B C^-1):  W = B C^-1, Ri12 = -A^-1 W
    double* Ri12 = Ri + (size_t)64 * 128;
    gemm(h, false, false, 64, 64, 64, 1.0, R11 + (size_t)64 * ldr, ldr, Ri22, 128, 0.0, W, 64, s,
         pred, kProfSampleUpd);
    gemm(h, false, false, 64, 64, 64, -1.0, Ri, 128, W, 64, 0.0, Ri12, 128, s, pred,
         kProfSampleUpd);
    gemm(h, false, false, 128, 128, 128, 1.0, S, lds, Ri, 128, 0.0, M, 128, s, pred,
         kProfSampleUpd);
    if (n2 > 0) {
      copy2d(S + (size_t)b * lds, lds, Bnew, ldb, ell, n2, s, pred);
      if (!rank_update(h, b, n2, b, M, b, R12, ldr, Bnew, ldb, s, pred, kProfSampleUpd))
        gemm(h, false, false, b, n2, b, -1.0, M, b, R12, ldr, 1.0, Bnew, ldb, s, pred,
             kProfSampleUpd);
    }
    return;
  }
  if (b == 16 || b == 32 || b == 64) {
    const int blocks = (int)std::max<int64_t>(1, (n2 + 127) / 128);
    ProfScope prof(h, kProfSampleUpd, 3.0 * b * b * n2, 8.0 * (2 * ell * n2 + b * b), s);
    count_launch();
    const double th = kEps34 * frob;
    const int ab = abort_on_degenerate ? 1 : 0;
    const size_t dsm = (size_t)(2 * b * b + b) * 8;
    kernel_attr((const void*)sample_update_reg_kernel<64>,
                cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    if (b == 16)
      sample_update_reg_kernel<16><<<blocks, 128, dsm, s>>>((int)ell, n2, S, lds, R11, R12, ldr,
                                                            th, Bnew, ldb, st, ab, i0);
    else if (b == 32)
      sample_update_reg_kernel<32><<<blocks, 128, dsm, s>>>((int)ell, n2, S, lds, R11, R12, ldr,
                                                            th, Bnew, ldb, st, ab, i0);
    else
      sample_update_reg_kernel<64><<<blocks, 128, dsm, s>>>((int)ell, n2, S, lds, R11, R12, ldr,
                                                            th, Bnew, ldb, st, ab, i0);
    RQ_CHECK_LAUNCH();
    return;
  }
  size_t smem = ((size_t)b * b + (size_t)b * kSuThreads) * 8;
  const bool staged = smem <= h.smem_optin;
  if (!staged) smem = (size_t)b * kSuThreads * 8;
  kernel_attr((const void*)sample_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)std::max<size_t>(smem, 48 * 1024));
  if (smem > h.smem_optin) throw InvalidArg("sample update block too wide");
  const int blocks = (int)std::max<int64_t>(1, (n2 + kSuThreads - 1) / kSuThreads);
  ProfScope prof(h, kProfSampleUpd, 3.0 * b * b * n2, 8.0 * (2 * ell * n2 + b * b), s);
  count_launch();
  sample_update_kernel<<<blocks, kSuThreads, smem, s>>>(
      (int)ell, (int)b, n2, S, lds, R11, R12, ldr, kEps34 * frob, Bnew, ldb, st,
      abort_on_degenerate ? 1 : 0, i0, staged ? 1 : 0);
  RQ_CHECK_LAUNCH();
}

void apply_swaps(Handle& h, const int64_t* piv, int64_t got_max, int64_t i0,
                 const SwapTargets& t, Status* st, cudaStream_t s) {
  if (got_max > 256) throw InvalidArg("at most 256 pivots per block");
  ProfScope prof(h, kProfSwap, 0.0, 32.0 * got_max * t.m, s);
  const int uw = (int)((t.m + kSwapRows - 1) / kSwapRows);
  const int ur = t.Rf ? (int)((t.rf_rows + kSwapRows - 1) / kSwapRows) : 0;
  const int uf = t.Wf ? (int)((t.wf_cols + kSwapRows - 1) / kSwapRows) : 0;
  const size_t smem = (size_t)2 * got_max * kSwapRows * 8;
  kernel_attr((const void*)swap_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)std::max<size_t>(smem, 48 * 1024));
  swap_fused_kernel<<<std::max(uw + ur + uf, 1), 256, smem, s>>>(piv, i0, t, st, uw, ur);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void column_norms(Handle& h, const double* A, int64_t m, int64_t n, int64_t lda, bool sequential,
                  double* out, cudaStream_t s) {
  if (n <= 0) return;
  if (m > 0x7fffffff) throw InvalidArg("column_norms: too many rows");
  ProfScope prof(h, kProfMisc, 2.0 * m * n, 8.0 * m * n, s);
  col_norms_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A, m, n, lda, sequential ? 1 : 0,
                                                               out);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void frob_norm(Handle& h, const double* A, int64_t m, int64_t n, int64_t lda, double* out,
               cudaStream_t s) {
  double* part = (double*)h.buf("frob_part", kNormBlocks * 8, s);
  sumsq_partial_kernel<<<kNormBlocks, kNormThreads, 0, s>>>(A, m, n, lda, part);
  RQ_CHECK_LAUNCH();
  count_launch();
  sumsq_final_kernel<<<1, 32, 0, s>>>(part, out);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
            int64_t cols, cudaStream_t s, const Status* st) {
  if (rows <= 0 || cols <= 0) return;
  copy2d_kernel<<<grid_for(rows * cols, 148), 256, 0, s>>>(src, lds, dst, ldd, rows, cols, st);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void downdate_norms(const double* norms, const double* row, int64_t inc, int64_t n,
                    const double* orig_sq, double guard, double* out, int32_t* unsafe,
                    cudaStream_t s) {
  if (n <= 0) return;
  norm_downdate_kernel<<<grid_for(n, 148), 256, 0, s>>>(norms, row, inc, n, orig_sq, guard, out,
                                                       unsafe);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void halves_guard(Handle& h, double* work, int64_t ldw, int64_t mm, int64_t cols, Status* st,
                  bool restore, int64_t i0, double* Y, int64_t ldy, double* tau, cudaStream_t s) {
  double* snap = (double*)h.buf("halves_snap", (size_t)mm * cols * 8, s);
  int64_t* sst = (int64_t*)h.buf("halves_sst", 16, s);
  halves_guard_kernel<<<grid_for(mm * cols, 148), 256, 0, s>>>(work, ldw, mm, cols, snap, sst, st,
                                                               restore ? 1 : 0, i0, Y, ldy, tau);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void fill2d(double* dst, int64_t ldd, int64_t rows, int64_t cols, double v, cudaStream_t s,
            const Status* st) {
  if (rows <= 0 || cols <= 0) return;
  fill2d_kernel<<<grid_for(rows * cols, 148), 256, 0, s>>>(dst, ldd, rows, cols, v, st);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void set_identity(double* dst, int64_t ldd, int64_t rows, int64_t cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  identity_kernel<<<grid_for(rows * cols, 148), 256, 0, s>>>(dst, ldd, rows, cols);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void transpose(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
               int64_t cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(src, lds, dst, ldd, rows, cols);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void scatter_cols(const double* src, int64_t lds, const int64_t* perm, double* dst,
                  int64_t ldd, int64_t rows, int64_t cols, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  scatter_cols_kernel<<<grid_for(rows * cols, 148), 256, 0, s>>>(src, lds, perm, dst, ldd,
                                                                  rows, cols);
  RQ_CHECK_LAUNCH();
  count_launch();
}

void t_factor(Handle& h, const double* Y, int64_t ldy, int64_t mm, int64_t nb,
              const double* tau, double* T, int64_t ldt, cudaStream_t s, const Status* st) {
  if (nb <= 0) return;
  double* G = (double*)h.buf("tf_gram", (size_t)nb * nb * 8, s);
  gemm(h, true, false, nb, nb, mm, 1.0, Y, ldy, Y, ldy, 0.0, G, nb, s, st, kProfPanel);
  if (nb <= 64 && h.t_inverse) {
    constexpr size_t kInvSmem = 3 * 64 * 65 * 8;
    kernel_attr((const void*)t_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)kInvSmem);
    ProfScope prof(h, kProfPanel, (double)nb * nb * nb / 3.0, 16.0 * nb * nb, s);
    t_inverse_kernel<<<1, 256, kInvSmem, s>>>(G, nb, tau, (int)nb, T, ldt, st);
    RQ_CHECK_LAUNCH();
    count_launch();
    return;
  }
  const size_t smem = nb <= 128 ? ((size_t)nb * nb + nb) * 8 : (size_t)nb * 8;
  kernel_attr((const void*)t_recurrence_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)std::max<size_t>(smem, 48 * 1024));
  ProfScope prof(h, kProfPanel, (double)nb * nb * nb / 3.0, 16.0 * nb * nb, s);
  t_recurrence_kernel<<<1, 256, smem, s>>>(G, nb, tau, (int)nb, T, ldt, st);
  RQ_CHECK_LAUNCH();
  count_launch();
}

}  // namespace rq
