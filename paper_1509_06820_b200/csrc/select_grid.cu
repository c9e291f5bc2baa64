// K4 (grid variant, wide samples): pivot-block selection = `want` greedy steps of column-pivoted
// Householder QR on the small (b+p) x nt Gaussian sample, in one persistent
// cooperative kernel (randomized.py:85-104 -> qrcp.py:63-84, NormTracker
// kernels.py:196-233, form/apply_reflector kernels.py:26-56).
//
// Layout: the sample's columns are dealt out to P CTAs in contiguous chunks
// and stay resident in shared memory (global/L2 fallback when a chunk does
// not fit).  Columns never move: a swap only relabels logical positions, so
// a step costs one grid barrier:
//   publish local best (norm, position) + that column's data
//   -> barrier -> every CTA reduces the P candidates identically
//   -> forms the reflector redundantly (bit-identical in every CTA)
//   -> applies it to its own active columns, downdates their norms with the
//      sqrt(eps) recompute guard, and publishes its next candidate.
// Ties break to the lowest logical position (np.argmax first-max semantics).
// Initial norms use numpy's pairwise summation, so they are bit-identical to
// np.linalg.norm(B, axis=0).
#include "runtime.hpp"

namespace rq {

namespace {

constexpr int kSelThreads = 256;

struct SelGridArgs {
  int ell, nt, want;
  int abort_on_short;
  int64_t i0;
  const double* B; int64_t ldb;
  double* S; int64_t lds;
  int64_t* piv;
  double* Ys; int64_t ldys;
  double* taus;
  Status* st;
  unsigned int* bar;
  double* pubval;   // [2][P]
  int* pubpos;      // [2][P]
  double* pubcol;   // [2][P][ell]
  double* pubsq;    // [P]
  double* gstore;   // fallback column store
  int cpb, ldl, use_smem;
};

struct Cand {
  double val;
  int pos;   // logical position (tie-break: lowest wins)
  int idx;   // local column (publish) or owner CTA (global reduce)
};
RQ_DEV bool better(const Cand& a, const Cand& b) {
  return a.val > b.val || (a.val == b.val && a.pos < b.pos);
}
RQ_DEV Cand warp_best(Cand c) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    Cand o;
    o.val = __shfl_xor_sync(0xffffffffu, c.val, off);
    o.pos = __shfl_xor_sync(0xffffffffu, c.pos, off);
    o.idx = __shfl_xor_sync(0xffffffffu, c.idx, off);
    if (better(o, c)) c = o;
  }
  return c;
}
RQ_DEV double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}
// sum over an aligned group of 8 lanes; every lane of the group gets the same value
RQ_DEV double group8_sum(double v, unsigned mask) {
#pragma unroll
  for (int off = 4; off; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(mask, v, off, 8));
  return v;
}

constexpr int kNoPos = 0x7fffffff;

__global__ void __launch_bounds__(kSelThreads, 1) select_grid_kernel(SelGridArgs a) {
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSelThreads / 32;
  constexpr int NG = kSelThreads / 8;  // 8-lane column groups
  const int grp = tid >> 3, gl = tid & 7;
  const unsigned gmask = 0xffu << (lane & 24);  // the 8 lanes of my group
  const int P = gridDim.x, me = blockIdx.x;
  const int ell = a.ell, ldl = a.ldl;
  const int c0 = me * a.cpb;
  const int ncol = max(0, min(a.nt - c0, a.cpb));

  double* store = a.use_smem ? sm : a.gstore + (size_t)me * a.cpb * ldl;
  double* meta = a.use_smem ? sm + (size_t)a.cpb * ldl : sm;
  double* nrm = meta;                 // [cpb]
  double* orig = nrm + a.cpb;         // [cpb]
  double* xb = orig + a.cpb;          // [ell] pivot column
  double* vb = xb + ell;              // [ell] v
  double* tvb = vb + ell;             // [ell] tau*v
  double* wv = tvb + ell;             // [NW + 8] scratch
  int* pos = (int*)(wv + NW + 8);     // [cpb]
  __shared__ Cand s_red[NW];
  __shared__ double s_sc[8];
  __shared__ Cand s_win;
  __shared__ int s_lc[2];             // local column of the candidate published per parity
  __shared__ double s_sq[160];

  unsigned int epoch = 0;

  // ---- load my columns, initial norms (pairwise, bit-identical to numpy)
  {
    const int total = ncol * ell;
#pragma unroll 4
    for (int e = tid; e < total; e += kSelThreads) {
      const int c = e / ell, i = e - c * ell;
      store[(size_t)c * ldl + i] = a.B[(size_t)(c0 + c) * a.ldb + i];
    }
  }
  __syncthreads();
  double mysq = 0.0;  // fixed-order per-thread partial of ||B||_F^2
  for (int c = tid; c < ncol; c += kSelThreads) {
    const double sq = pairwise_sumsq(store + (size_t)c * ldl, ell, 1);
    const double nv = sqrt(sq);
    nrm[c] = nv;
    orig[c] = __dmul_rn(nv, nv);
    pos[c] = c0 + c;
    mysq = __dadd_rn(mysq, sq);
  }
  {
    double v = warp_sum(mysq);
    if (lane == 0) wv[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t = __dadd_rn(t, wv[w]);
      a.pubsq[me] = t;
    }
  }

  // local argmax over active columns (position >= jstart); publishes the
  // candidate (value, position) and its column into parity slot `par`
  auto publish = [&](int jstart, int par) {
    Cand best{-1.0, kNoPos, -1};
    for (int c = tid; c < ncol; c += kSelThreads) {
      if (pos[c] >= jstart) {
        Cand cc{nrm[c], pos[c], c};
        if (better(cc, best)) best = cc;
      }
    }
    best = warp_best(best);
    if (lane == 0) s_red[warp] = best;
    __syncthreads();
    if (warp == 0) {
      Cand b = lane < NW ? s_red[lane] : Cand{-1.0, kNoPos, -1};
      b = warp_best(b);
      if (lane == 0) {
        s_lc[par] = b.idx;
        a.pubval[par * P + me] = b.val;
        a.pubpos[par * P + me] = b.pos;
      }
    }
    __syncthreads();
    const int lc = s_lc[par];
    if (lc >= 0)
      for (int i = tid; i < ell; i += kSelThreads)
        a.pubcol[((size_t)par * P + me) * ell + i] = store[(size_t)lc * ldl + i];
  };

  publish(0, 0);
  grid_barrier(a.bar, epoch);

  // tol = eps * ||B||_F  (randomized.py:98), same summation order everywhere
  for (int q = tid; q < P; q += kSelThreads) s_sq[q] = a.pubsq[q];
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < P; ++q) t = __dadd_rn(t, s_sq[q]);
    s_sc[0] = kEps * sqrt(t);
  }
  __syncthreads();
  const double tol = s_sc[0];

  int got = a.want;
  int64_t l2 = 0, l2b = 0;
  for (int j = 0; j < a.want; ++j) {
    const int par = j & 1;
    // ---- global argmax over the P candidates (total order -> identical everywhere)
    {
      Cand best{-1.0, kNoPos, -1};
      for (int q = tid; q < P; q += kSelThreads) {
        Cand cc{a.pubval[par * P + q], a.pubpos[par * P + q], q};
        if (cc.pos != kNoPos && better(cc, best)) best = cc;
      }
      best = warp_best(best);
      if (lane == 0) s_red[warp] = best;
      __syncthreads();
      if (warp == 0) {
        Cand b = lane < NW ? s_red[lane] : Cand{-1.0, kNoPos, -1};
        b = warp_best(b);
        if (lane == 0) s_win = b;
      }
      __syncthreads();
    }
    const Cand win = s_win;
    const int p = win.pos, owner = win.idx;
    if (owner < 0 || !(win.val > tol)) {  // max trailing norm <= tol: halt (qrcp.py:69-71)
      got = j;
      break;
    }
    // ---- fetch the pivot column, relabel positions (swap j <-> p)
    for (int i = tid; i < ell; i += kSelThreads)
      xb[i] = a.pubcol[((size_t)par * P + owner) * ell + i];
    const int lc_piv = s_lc[par];
    for (int c = tid; c < ncol; c += kSelThreads)
      if (pos[c] == j && p != j) pos[c] = p;
    __syncthreads();
    // ---- reflector from x[j:] (kernels.py:26-44), identical in every CTA
    if (warp == 0) {
      double sq = 0.0;
      for (int i = j + lane; i < ell; i += 32) sq = __fma_rn(xb[i], xb[i], sq);
      sq = warp_sum(sq);
      if (lane == 0) {
        const double norm = sqrt(sq);
        const double alpha = xb[j];
        double beta = 0.0, tau = 0.0, den = 1.0;
        if (norm != 0.0) {
          beta = alpha >= 0.0 ? -norm : norm;
          den = __dsub_rn(alpha, beta);
          tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
        }
        s_sc[2] = beta; s_sc[3] = tau; s_sc[4] = den; s_sc[5] = norm;
      }
    }
    __syncthreads();
    const double beta = s_sc[2], tau = s_sc[3], den = s_sc[4];
    const bool zero = s_sc[5] == 0.0;
    for (int i = j + tid; i < ell; i += kSelThreads) {
      const double v = (i == j) ? 1.0 : (zero ? xb[i] : __ddiv_rn(xb[i], den));
      vb[i] = v;
      tvb[i] = __dmul_rn(tau, v);
    }
    if (owner == me) {
      if (tid == 0) pos[lc_piv] = j;
      // pivot column: rows < j keep R, row j = beta, below = 0 (qrcp.py:80-81)
      for (int i = j + tid; i < ell; i += kSelThreads)
        store[(size_t)lc_piv * ldl + i] = (i == j) ? beta : 0.0;
    }
    if (me == 0 && tid == 0) {
      a.piv[j] = p;
      if (a.taus) a.taus[j] = tau;
      const int64_t cols = (int64_t)a.nt - j - 1;
      if (tau != 0.0 && cols > 0) {
        l2 += 4LL * (ell - j) * cols;
        l2b += 16LL * (ell - j) * cols;
      }
    }
    __syncthreads();
    if (me == 0 && a.Ys)
      for (int i = tid; i < ell; i += kSelThreads)
        a.Ys[(size_t)j * a.ldys + i] = i < j ? 0.0 : vb[i];
    // ---- apply H_j to my active columns (pos > j) and downdate their norms;
    //      one 8-lane group per column
    for (int c = grp; c < ncol; c += NG) {
      if (pos[c] <= j) continue;  // uniform within the group
      double* col = store + (size_t)c * ldl;
      if (tau != 0.0) {
        double d = 0.0;
        for (int i = j + gl; i < ell; i += 8) d = __fma_rn(vb[i], col[i], d);
        const double w = group8_sum(d, gmask);
        for (int i = j + gl; i < ell; i += 8) col[i] = __dsub_rn(col[i], __dmul_rn(tvb[i], w));
      }
      if (j + 1 < a.nt) {
        // NormTracker.downdate with row j of the updated sample (kernels.py:222-233)
        __syncwarp(gmask);
        const double row = col[j];
        const double nv = nrm[c];
        double nsq = __dsub_rn(__dmul_rn(nv, nv), __dmul_rn(row, row));
        nsq = nsq > 0.0 ? nsq : 0.0;
        if (!(nsq < __dmul_rn(kGuard, orig[c]))) {
          if (gl == 0) nrm[c] = sqrt(nsq);
        } else {
          double sq = 0.0;
          for (int i = j + 1 + gl; i < ell; i += 8) sq = __fma_rn(col[i], col[i], sq);
          sq = group8_sum(sq, gmask);
          const double fresh = sqrt(sq);
          if (gl == 0) { nrm[c] = fresh; orig[c] = __dmul_rn(fresh, fresh); }
        }
      }
    }
    __syncthreads();
    publish(j + 1, par ^ 1);
    grid_barrier(a.bar, epoch);
  }

  // ---- write the transformed sample in pivoted order
  {
    const int total = ncol * ell;
    for (int e = tid; e < total; e += kSelThreads) {
      const int c = e / ell, i = e - c * ell;
      a.S[(size_t)pos[c] * a.lds + i] = store[(size_t)c * ldl + i];
    }
  }
  if (me == 0 && tid == 0) {
    a.st->got = got;
    a.st->level2 += l2;
    a.st->l2bytes += l2b;
    if (a.abort_on_short && got < a.want) {
      a.st->abort_i0 = a.i0;
      __threadfence();
      a.st->abort = kAbortShortSample;
    }
  }
}

}  // namespace

void select_pivots_grid(Handle& h, int64_t ell, int64_t nt, int64_t want, const double* B,
                   int64_t ldb, const SelectOut& out, Status* st, bool abort_on_short,
                   int64_t i0, cudaStream_t s) {
  if (want < 1 || want > std::min(ell, nt))
    throw InvalidArg("cannot select " + std::to_string(want) + " pivots from a " +
                     std::to_string(ell) + " x " + std::to_string(nt) + " sample");
  // CTA count: >= 32 columns per CTA, at most one CTA per SM
  int P = (int)std::min<int64_t>(h.num_sms, (nt + 31) / 32);
  P = std::max(P, 1);
  const int cpb = (int)((nt + P - 1) / P);
  P = (int)((nt + cpb - 1) / cpb);
  const int ldl = (int)(ell | 1);
  const size_t meta = (size_t)(2 * cpb + 3 * ell + 8 + 8) * 8 + (size_t)(cpb + 8) * 4 + 64;
  if (P > 160) throw InvalidArg("select: too many CTAs");
  const size_t store = (size_t)cpb * ldl * 8;
  const bool use_smem = store + meta <= h.smem_optin - 2048;
  const size_t smem = (use_smem ? store : 0) + meta;
  SelGridArgs a{};
  a.ell = (int)ell; a.nt = (int)nt; a.want = (int)want;
  a.abort_on_short = abort_on_short ? 1 : 0;
  a.i0 = i0;
  a.B = B; a.ldb = ldb;
  a.S = out.S; a.lds = out.lds; a.piv = out.piv; a.Ys = out.Ys; a.ldys = out.ldys;
  a.taus = out.taus;
  a.st = st;
  a.bar = (unsigned int*)h.buf("selg_bar", 64, s);
  a.pubval = (double*)h.buf("selg_pubval", (size_t)2 * P * 8, s);
  a.pubpos = (int*)h.buf("selg_pubpos", (size_t)2 * P * 4, s);
  a.pubcol = (double*)h.buf("selg_pubcol", (size_t)2 * P * ell * 8, s);
  a.pubsq = (double*)h.buf("selg_pubsq", (size_t)P * 8, s);
  a.gstore = use_smem ? nullptr : (double*)h.buf("selg_gstore", (size_t)P * store, s);
  a.cpb = cpb; a.ldl = ldl; a.use_smem = use_smem ? 1 : 0;
  RQ_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
  static size_t attr = 0;
  if (smem > attr) {
    RQ_CUDA(cudaFuncSetAttribute(select_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 48 * 1024)));
    attr = std::max<size_t>(smem, 48 * 1024);
  }
  void* args[] = {&a};
  ProfScope prof(h, kProfSelect, 4.0 * ell * nt * want, 16.0 * ell * nt, s);
  count_launch();
  RQ_CUDA(cudaLaunchCooperativeKernel((void*)select_grid_kernel, dim3(P), dim3(kSelThreads), args,
                                      smem, s));
}

}  // namespace rq
