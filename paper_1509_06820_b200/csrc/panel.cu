// K5: panel Householder QR + _panel_rank + T factor in ONE thread-block
// cluster (qrcp.py:206-219 panel_householder; randomized.py:150-155
// _panel_rank; kernels.py:139-147 build_t_matrix).
//
// The mm x bw panel is split by rows over the Q <= 16 CTAs of a cluster and
// kept in shared memory (global/L2 fallback when a row slab does not fit).
// Per column j every CTA publishes, in its own shared memory, the partial
// inner products d_c = sum_{r>j} P[r,j] P[r,c] over its rows (d_j is the
// partial squared norm; the owner of row j also publishes that row), then a
// cluster barrier (~0.23 us on B200, 5x cheaper than a grid barrier), then
// every CTA reads the Q partial vectors over DSMEM and reduces them in the
// same fixed order -- so beta, tau and w are bit-identical in every CTA -- and
// updates its rows:
//   P[r,c] -= (tau v_r) w_c,   v_r = P[r,j] / (alpha - beta)   (kernels.py:42,52)
// fused with the partials of column j+1 (one pass over the slab per column).
// Reflector convention is the reference's: beta = -sign(alpha)||x||,
// sign(0) = +1, a nonzero column is always reflected, a zero column gives
// tau = 0.  v is kept below the diagonal until the commit, which writes R
// (zeros below the diagonal) and the unit-lower Y only when the policy
// allows it (speculative path: all columns usable, else Status.abort).
// Using 16 SMs also leaves the rest of the GPU free for concurrent GEMMs.
#include <cooperative_groups.h>

#include "runtime.hpp"

namespace cg = cooperative_groups;

namespace rq {

namespace {

constexpr int kPanThreads = 256;
constexpr int kMaxBw = 256;
constexpr int kMaxCluster = 16;

struct PanArgs {
  int64_t mm;
  int bw;
  const double* P; int64_t ldp;
  double* Rdst; int64_t ldr; int64_t rrows;
  double* Y; int64_t ldy;
  double* tau;
  double* T; int64_t ldt;
  double tol;
  int policy;
  int raise_abort;
  int64_t i0;
  Status* st;
  double* gstore;     // spill columns (global/L2), [Q][bw - ncs][ldl]
  int rpb, ldl, ncs, cs;  // ncs = leading columns kept in shared memory
};

__global__ void __launch_bounds__(kPanThreads, 1) panel_kernel(PanArgs a) {
  if (aborted(a.st)) return;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int Q = (int)cluster.num_blocks(), me = (int)cluster.block_rank();
  const int bw = a.bw, cs = a.cs, groups = kPanThreads / cs;
  const int tc = tid % cs, tg = tid / cs;
  const int64_t r0 = (int64_t)me * a.rpb;
  const int nrow = (int)imax64(0, imin64(a.mm - r0, a.rpb));
  const int ldl = a.ldl;
  const int npair = bw * (bw - 1) / 2;
  const int ncs = a.ncs;
  double* gsp = a.gstore ? a.gstore + (size_t)me * (bw - ncs) * ldl : nullptr;
  // column c of my row slab: shared memory for c < ncs, else the L2 spill
  auto colp = [&](int c) -> double* {
    return c < ncs ? sm + (size_t)c * ldl : gsp + (size_t)(c - ncs) * ldl;
  };
  double* aux = sm + (size_t)ncs * ldl;
  double* xpub = aux;                      // [2][2*bw] DSMEM-published partials + row
  double* part = xpub + 4 * bw;            // [groups][bw]
  double* dsum = part + groups * bw;       // [bw]
  double* rowj = dsum + bw;                // [bw]
  double* wsh = rowj + bw;                 // [bw]
  double* taus = wsh + bw;                 // [bw]
  double* tvrow = taus + bw;               // [rpb]  tau * v_r for my rows
  double* xnext = tvrow + a.rpb;           // [rpb]  updated column j+1
  double* gpart = xnext + a.rpb;           // [npair] Gram partial
  double* gfin = gpart + npair;            // [npair] reduced Gram (rank 0)
  __shared__ double s_sc[4];
  __shared__ int s_usable;
  const int stride = 2 * bw;
  const int64_t ncols = imin64(bw, a.mm);

  // ---- load my row slab (coalesced down each column, many loads in flight)
  {
    const int total = nrow * bw;
#pragma unroll 8
    for (int e = tid; e < total; e += kPanThreads) {
      const int c = e / nrow, r = e - c * nrow;
      colp(c)[r] = a.P[(size_t)c * a.ldp + r0 + r];
    }
  }
  if (tid == 0) s_usable = (int)ncols;
  __syncthreads();

  // partials of column 0 over my rows r > 0 (+ row 0 if owned) -> xpub[0]
  {
    const int rstart = r0 == 0 ? 1 : 0;
    const double* x0 = colp(0);
    for (int c = tc; c < bw; c += cs) {
      const double* col = colp(c);
      double d = 0.0;
      for (int r = rstart + tg; r < nrow; r += groups) d = __fma_rn(x0[r], col[r], d);
      part[tg * bw + c] = d;
    }
    __syncthreads();
    if (tg == 0)
      for (int c = tc; c < bw; c += cs) {
        double d = part[c];
        for (int g = 1; g < groups; ++g) d = __dadd_rn(d, part[g * bw + c]);
        xpub[c] = d;
      }
    if (r0 == 0 && nrow > 0)
      for (int c = tid; c < bw; c += kPanThreads) xpub[bw + c] = colp(c)[0];
  }

  int64_t l2 = 0, l2b = 0;
  for (int j = 0; j < ncols; ++j) {
    cluster.sync();
    const int par = j & 1;
    const int owner = (int)(j / a.rpb);
    // (1) reduce the Q partial vectors over DSMEM in fixed q order
    for (int c = j + tid; c < bw; c += kPanThreads) {
      double v[kMaxCluster];
#pragma unroll
      for (int q = 0; q < kMaxCluster; ++q)
        if (q < Q) v[q] = cluster.map_shared_rank(xpub, q)[par * stride + c];
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxCluster; ++q)
        if (q < Q) d = __dadd_rn(d, v[q]);
      dsum[c] = d;
      rowj[c] = cluster.map_shared_rank(xpub, owner)[par * stride + bw + c];
    }
    __syncthreads();
    // (2) reflector scalars (kernels.py:35-44), identical in every CTA
    if (tid == 0) {
      const double alpha = rowj[j];
      const double norm = sqrt(__fma_rn(alpha, alpha, dsum[j]));
      double beta = 0.0, tau = 0.0, den = 1.0;
      if (norm != 0.0) {
        beta = alpha >= 0.0 ? -norm : norm;
        den = __dsub_rn(alpha, beta);
        tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
      }
      s_sc[0] = beta; s_sc[1] = tau; s_sc[2] = den; s_sc[3] = norm;
      taus[j] = tau;
      if (s_usable == ncols && fabs(beta) <= a.tol) s_usable = j;  // _panel_rank
      if (me == 0) {
        const int64_t cols = bw - j - 1;
        if (tau != 0.0 && cols > 0) {
          l2 += 4 * (a.mm - j) * cols;
          l2b += 16 * (a.mm - j) * cols;
        }
      }
    }
    __syncthreads();
    const double beta = s_sc[0], tau = s_sc[1], den = s_sc[2];
    const bool zero = s_sc[3] == 0.0;
    // (3) w_c = P[j,c] + (sum_{r>j} x_r P[r,c]) / (alpha - beta); v_r once per row
    for (int c = j + 1 + tid; c < bw; c += kPanThreads)
      wsh[c] = zero ? rowj[c] : __dadd_rn(rowj[c], __ddiv_rn(dsum[c], den));
    const int rj = (int)imax64(0, (int64_t)j - r0);  // first local row >= j
    {
      double* xj = colp(j);
      for (int r = rj + tid; r < nrow; r += kPanThreads) {
        const bool diag = r0 + r == j;
        const double v = diag ? 1.0 : (zero ? xj[r] : __ddiv_rn(xj[r], den));
        tvrow[r] = __dmul_rn(tau, v);
        xj[r] = diag ? beta : v;
      }
    }
    __syncthreads();
    if (j + 1 >= ncols) break;
    // (4) updated column j+1 first (it feeds the next partials)
    {
      const double w1 = wsh[j + 1];
      double* x1 = colp(j + 1);
      for (int r = rj + tid; r < nrow; r += kPanThreads) {
        const double nv = tau != 0.0 ? __dsub_rn(x1[r], __dmul_rn(tvrow[r], w1)) : x1[r];
        x1[r] = nv;
        xnext[r] = nv;
      }
    }
    __syncthreads();
    // (5) fused trailing update of columns > j+1 and the partials of step j+1
    {
      const int rs1 = (int)imax64(0, (int64_t)j + 2 - r0);  // rows > j+1
      for (int c = j + 1 + tc; c < bw; c += cs) {
        double* col = colp(c);
        double d = 0.0;
        if (c == j + 1) {
          for (int r = rs1 + tg; r < nrow; r += groups) d = __fma_rn(xnext[r], xnext[r], d);
        } else {
          const double w = wsh[c];
          for (int r = rj + tg; r < nrow; r += groups) {
            const double nv = tau != 0.0 ? __dsub_rn(col[r], __dmul_rn(tvrow[r], w)) : col[r];
            col[r] = nv;
            if (r >= rs1) d = __fma_rn(xnext[r], nv, d);
          }
        }
        part[tg * bw + c] = d;
      }
      __syncthreads();
      double* out = xpub + (size_t)((j + 1) & 1) * stride;
      if (tg == 0)
        for (int c = j + 1 + tc; c < bw; c += cs) {
          double d = part[c];
          for (int g = 1; g < groups; ++g) d = __dadd_rn(d, part[g * bw + c]);
          out[c] = d;
        }
      if (j + 1 >= r0 && j + 1 < r0 + nrow) {
        const int lr = (int)(j + 1 - r0);
        for (int c = j + 1 + tid; c < bw; c += kPanThreads) out[bw + c] = colp(c)[lr];
      }
    }
  }
  cluster.sync();  // every CTA is done reading the others' partials

  // ---- commit
  const int usable = s_usable;
  int ncommit;
  if (a.policy == kPanelCommitIfFull) ncommit = usable == ncols ? (int)ncols : 0;
  else if (a.policy == kPanelCommitUsable) ncommit = usable;
  else ncommit = (int)ncols;
  if (me == 0 && tid == 0) {
    a.st->usable = usable;
    a.st->level2 += l2;
    a.st->l2bytes += l2b;
    if (a.raise_abort && usable < ncols) {
      a.st->abort_i0 = a.i0;
      __threadfence();
      a.st->abort = kAbortPanelRank;
    }
  }
  if (ncommit == 0) return;  // uniform across the cluster
  {
    const int total = nrow * ncommit;
#pragma unroll 4
    for (int e = tid; e < total; e += kPanThreads) {
      const int c = e / nrow, r = e - c * nrow;
      const int64_t gr = r0 + r;
      const double val = colp(c)[r];
      a.Y[(size_t)c * a.ldy + gr] = gr < c ? 0.0 : (gr == c ? 1.0 : val);
      if (gr < a.rrows) a.Rdst[(size_t)c * a.ldr + gr] = gr <= c ? val : 0.0;
    }
  }
  if (me == 0)
    for (int c = tid; c < ncommit; c += kPanThreads) a.tau[c] = taus[c];
  if (a.T == nullptr) return;

  // ---- T factor (kernels.py:139-147): Gram G = Y^T Y (strict upper) from
  // per-CTA partials reduced over DSMEM, then on rank 0
  // T[:j,j] = -tau_j T[:j,:j] G[:j,j]
  const int nc = ncommit;
  const int np = nc * (nc - 1) / 2;
  for (int e = tid; e < np; e += kPanThreads) {
    int j = (int)((1.0 + sqrt(1.0 + 8.0 * e)) * 0.5);
    while (j * (j - 1) / 2 > e) --j;
    while ((j + 1) * j / 2 <= e) ++j;
    const int i = e - j * (j - 1) / 2;
    const int rs = (int)imax64(0, (int64_t)j - r0);  // rows >= j carry both
    const double* yi = colp(i);
    const double* yj = colp(j);
    double g = 0.0;
    for (int r = rs; r < nrow; ++r) g = __fma_rn(yi[r], (r0 + r == j) ? 1.0 : yj[r], g);
    gpart[e] = g;
  }
  cluster.sync();
  {
    // this CTA reduces a slice of the pair list into rank 0's gfin
    const int per = (np + Q - 1) / Q;
    const int lo = me * per, hi = min(np, lo + per);
    double* g0 = cluster.map_shared_rank(gfin, 0);
    for (int e = lo + tid; e < hi; e += kPanThreads) {
      double g = 0.0;
      for (int q = 0; q < Q; ++q) g = __dadd_rn(g, cluster.map_shared_rank(gpart, q)[e]);
      g0[e] = g;
    }
  }
  cluster.sync();
  if (me != 0) return;
  // T workspace in the (now free) shared column store when it is big enough
  const bool tsm = (int64_t)ncs * ldl >= (int64_t)nc * nc;
  double* Tw = tsm ? sm : a.T;
  const int ldtw = tsm ? nc : (int)a.ldt;
  for (int e = tid; e < nc * nc; e += kPanThreads) Tw[(e % nc) + (size_t)(e / nc) * ldtw] = 0.0;
  __syncthreads();
  for (int j = 0; j < nc; ++j) {
    const double* gcol = gfin + j * (j - 1) / 2;  // G[0:j, j]
    for (int i = tid; i < j; i += kPanThreads) {
      double t = 0.0;
      for (int l = i; l < j; ++l) t = __fma_rn(Tw[i + (size_t)l * ldtw], gcol[l], t);
      wsh[i] = t;
    }
    __syncthreads();
    for (int i = tid; i < j; i += kPanThreads) Tw[i + (size_t)j * ldtw] = __dmul_rn(-taus[j], wsh[i]);
    if (tid == 0) Tw[j + (size_t)j * ldtw] = taus[j];
    __syncthreads();
  }
  if (tsm)
    for (int e = tid; e < nc * nc; e += kPanThreads) {
      const int i = e % nc, j = e / nc;
      a.T[i + (size_t)j * a.ldt] = Tw[i + (size_t)j * ldtw];
    }
}

}  // namespace

void panel_qr(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
              const PanelOut& out, double tol, PanelPolicy policy, bool raise_abort, Status* st,
              int64_t i0, cudaStream_t s) {
  if (bw < 1 || bw > kMaxBw) throw InvalidArg("panel width must be in [1, 256]");
  if (mm < 1) throw InvalidArg("panel needs at least one row");
  int Q = 1;
  while (Q < kMaxCluster && (int64_t)Q * 128 < mm) Q <<= 1;
  const int rpb = (int)((mm + Q - 1) / Q);
  int cs = 1;
  while (cs < bw && cs < kPanThreads) cs <<= 1;
  const int groups = kPanThreads / cs;
  const int ldl = rpb | 1;
  const size_t npair = (size_t)bw * (bw - 1) / 2;
  const size_t aux = ((size_t)4 * bw + (size_t)groups * bw + 5 * (size_t)bw + 2 * (size_t)rpb +
                      2 * npair + 8) * 8;
  if (aux > h.smem_optin - 2048) throw InvalidArg("panel too wide for shared memory");
  const size_t colbytes = (size_t)ldl * 8;
  const int ncs = (int)std::min<size_t>(bw, (h.smem_optin - 2048 - aux) / colbytes);
  const size_t smem = (size_t)ncs * colbytes + aux;
  PanArgs a{};
  a.mm = mm; a.bw = (int)bw; a.P = P; a.ldp = ldp;
  a.Rdst = out.Rdst; a.ldr = out.ldr; a.rrows = out.rrows;
  a.Y = out.Y; a.ldy = out.ldy; a.tau = out.tau; a.T = out.T; a.ldt = out.ldt;
  a.tol = tol; a.policy = (int)policy; a.raise_abort = raise_abort ? 1 : 0; a.i0 = i0;
  a.st = st;
  a.gstore = ncs < bw ? (double*)h.buf("pan_gstore", (size_t)Q * (bw - ncs) * colbytes, s)
                      : nullptr;
  a.rpb = rpb; a.ldl = ldl; a.ncs = ncs; a.cs = cs;
  static bool attr_init = false;
  static size_t attr = 0;
  if (!attr_init) {
    RQ_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_init = true;
  }
  if (smem > attr) {
    RQ_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 48 * 1024)));
    attr = std::max<size_t>(smem, 48 * 1024);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Q);
  cfg.blockDim = dim3(kPanThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = Q;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  ProfScope prof(h, kProfPanel, 2.0 * mm * bw * bw, 16.0 * mm * bw, s);
  count_launch();
  RQ_CUDA(cudaLaunchKernelEx(&cfg, panel_kernel, a));
}

}  // namespace rq
