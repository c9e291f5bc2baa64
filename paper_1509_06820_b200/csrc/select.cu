// K4: pivot-block selection = `want` greedy steps of column-pivoted
// Householder QR on the small (b+p) x nt Gaussian sample, in one persistent
// cooperative kernel (randomized.py:85-104 -> qrcp.py:63-84, NormTracker
// kernels.py:196-233, form/apply_reflector kernels.py:26-56).
//
// Layout: the sample's columns are dealt out to the P <= 16 CTAs of ONE
// thread-block cluster in contiguous chunks and stay resident in shared
// memory (columns beyond the shared-memory budget spill to global/L2).
// Columns never move: a swap only relabels logical positions, so a step costs
// one cluster barrier (~0.23 us on B200):
//   publish local best (norm, position) + that column's data in own smem
//   -> cluster barrier -> every CTA reads the P candidates over DSMEM and
//      reduces them identically
//   -> forms the reflector redundantly (bit-identical in every CTA)
//   -> applies it to its own active columns, downdates their norms with the
//      sqrt(eps) recompute guard, and publishes its next candidate.
// Ties break to the lowest logical position (np.argmax first-max semantics).
// Initial norms use numpy's pairwise summation, so they are bit-identical to
// np.linalg.norm(B, axis=0).
#include <cooperative_groups.h>

#include "runtime.hpp"

namespace cg = cooperative_groups;

namespace rq {

namespace {

constexpr int kSelThreads = 256;

constexpr int kMaxCluster = 16;

struct SelArgs {
  int ell, nt, want;
  int abort_on_short;
  int64_t i0;
  const double* B; int64_t ldb;
  double* S; int64_t lds;
  int64_t* piv;
  double* Ys; int64_t ldys;
  double* taus;
  Status* st;
  double* gstore;   // spill columns [P][cpb - ncs][ldl]
  int cpb, ldl, ncs;
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

__global__ void __launch_bounds__(kSelThreads, 1) select_kernel(SelArgs a) {
  if (aborted(a.st)) return;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSelThreads / 32;
  constexpr int NG = kSelThreads / 8;  // 8-lane column groups
  const int grp = tid >> 3, gl = tid & 7;
  const unsigned gmask = 0xffu << (lane & 24);  // the 8 lanes of my group
  const int P = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
  const int ell = a.ell, ldl = a.ldl, ncs = a.ncs;
  const int c0 = me * a.cpb;
  const int ncol = max(0, min(a.nt - c0, a.cpb));
  double* gsp = a.gstore ? a.gstore + (size_t)me * (a.cpb - ncs) * ldl : nullptr;
  auto colp = [&](int c) -> double* {
    return c < ncs ? sm + (size_t)c * ldl : gsp + (size_t)(c - ncs) * ldl;
  };
  double* meta = sm + (size_t)ncs * ldl;
  double* nrm = meta;                 // [cpb]
  double* orig = nrm + a.cpb;         // [cpb]
  double* xb = orig + a.cpb;          // [ell] pivot column
  double* vb = xb + ell;              // [ell] v
  double* tvb = vb + ell;             // [ell] tau*v
  double* ccol = tvb + ell;           // [2][ell] published candidate column (DSMEM)
  double* wv = ccol + 2 * ell;        // [NW + 8] scratch
  int* pos = (int*)(wv + NW + 8);     // [cpb]
  __shared__ Cand s_red[NW];
  __shared__ double s_sc[8];
  __shared__ Cand s_win;
  __shared__ int s_lc[2];             // local column of the published candidate
  __shared__ double s_cval[2];        // published candidate (DSMEM)
  __shared__ int s_cpos[2];
  __shared__ double s_sq;             // published ||B_local||^2 (DSMEM)

  // ---- load my columns, initial norms (pairwise, bit-identical to numpy)
  {
    const int total = ncol * ell;
#pragma unroll 4
    for (int e = tid; e < total; e += kSelThreads) {
      const int c = e / ell, i = e - c * ell;
      colp(c)[i] = a.B[(size_t)(c0 + c) * a.ldb + i];
    }
  }
  __syncthreads();
  double mysq = 0.0;  // fixed-order per-thread partial of ||B||_F^2
  for (int c = tid; c < ncol; c += kSelThreads) {
    const double sq = pairwise_sumsq(colp(c), ell, 1);
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
      s_sq = t;
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
        s_cval[par] = b.val;
        s_cpos[par] = b.pos;
      }
    }
    __syncthreads();
    const int lc = s_lc[par];
    if (lc >= 0) {
      const double* src = colp(lc);
      for (int i = tid; i < ell; i += kSelThreads) ccol[par * ell + i] = src[i];
    }
  };

  publish(0, 0);
  cluster.sync();

  // tol = eps * ||B||_F  (randomized.py:98), same summation order everywhere
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < P; ++q) t = __dadd_rn(t, *cluster.map_shared_rank(&s_sq, q));
    s_sc[0] = kEps * sqrt(t);
  }
  __syncthreads();
  const double tol = s_sc[0];

  int got = a.want;
  int64_t l2 = 0, l2b = 0;
  for (int j = 0; j < a.want; ++j) {
    const int par = j & 1;
    // ---- cluster-wide argmax over the P candidates (total order -> identical everywhere)
    if (warp == 0) {
      Cand b{-1.0, kNoPos, -1};
      if (lane < P) {
        const double v = cluster.map_shared_rank(s_cval, lane)[par];
        const int p = cluster.map_shared_rank(s_cpos, lane)[par];
        if (p != kNoPos) b = Cand{v, p, lane};
      }
      b = warp_best(b);
      if (lane == 0) s_win = b;
    }
    __syncthreads();
    const Cand win = s_win;
    const int p = win.pos, owner = win.idx;
    if (owner < 0 || !(win.val > tol)) {  // max trailing norm <= tol: halt (qrcp.py:69-71)
      got = j;
      break;
    }
    // ---- fetch the pivot column over DSMEM, relabel positions (swap j <-> p)
    {
      const double* oc = cluster.map_shared_rank(ccol, owner) + par * ell;
      for (int i = tid; i < ell; i += kSelThreads) xb[i] = oc[i];
    }
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
      double* pc = colp(lc_piv);
      for (int i = j + tid; i < ell; i += kSelThreads) pc[i] = (i == j) ? beta : 0.0;
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
      double* col = colp(c);
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
    cluster.sync();
  }

  // ---- write the transformed sample in pivoted order
  {
    const int total = ncol * ell;
    for (int e = tid; e < total; e += kSelThreads) {
      const int c = e / ell, i = e - c * ell;
      a.S[(size_t)pos[c] * a.lds + i] = colp(c)[i];
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
  cluster.sync();  // keep shared memory alive until every peer is done reading it
}

}  // namespace

void select_pivots(Handle& h, int64_t ell, int64_t nt, int64_t want, const double* B,
                   int64_t ldb, const SelectOut& out, Status* st, bool abort_on_short,
                   int64_t i0, cudaStream_t s) {
  if (want < 1 || want > std::min(ell, nt))
    throw InvalidArg("cannot select " + std::to_string(want) + " pivots from a " +
                     std::to_string(ell) + " x " + std::to_string(nt) + " sample");
  // cluster of P <= 16 CTAs, >= 32 columns each
  int P = 1;
  while (P < kMaxCluster && (int64_t)P * 32 < nt) P <<= 1;
  const int cpb = (int)((nt + P - 1) / P);
  const int ldl = (int)(ell | 1);
  const size_t meta = (size_t)(2 * cpb + 5 * ell + 8 + 8 + 8) * 8 + (size_t)(cpb + 8) * 4 + 256;
  if (meta > h.smem_optin - 2048) throw InvalidArg("select: sample too large");
  const size_t colbytes = (size_t)ldl * 8;
  const int ncs = (int)std::min<size_t>(cpb, (h.smem_optin - 2048 - meta) / colbytes);
  const size_t smem = (size_t)ncs * colbytes + meta;
  SelArgs a{};
  a.ell = (int)ell; a.nt = (int)nt; a.want = (int)want;
  a.abort_on_short = abort_on_short ? 1 : 0;
  a.i0 = i0;
  a.B = B; a.ldb = ldb;
  a.S = out.S; a.lds = out.lds; a.piv = out.piv; a.Ys = out.Ys; a.ldys = out.ldys;
  a.taus = out.taus;
  a.st = st;
  a.gstore = ncs < cpb ? (double*)h.buf("sel_gstore", (size_t)P * (cpb - ncs) * colbytes, s)
                       : nullptr;
  a.cpb = cpb; a.ldl = ldl; a.ncs = ncs;
  static bool attr_init = false;
  static size_t attr = 0;
  if (!attr_init) {
    RQ_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_init = true;
  }
  if (smem > attr) {
    RQ_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 48 * 1024)));
    attr = std::max<size_t>(smem, 48 * 1024);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(kSelThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = P;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  ProfScope prof(h, kProfSelect, 4.0 * ell * nt * want, 16.0 * ell * nt, s);
  count_launch();
  RQ_CUDA(cudaLaunchKernelEx(&cfg, select_kernel, a));
}

}  // namespace rq
