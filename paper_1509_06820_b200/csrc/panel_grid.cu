// K5 (grid variant, large panels): panel Householder QR + _panel_rank + T factor, one persistent
// cooperative kernel (qrcp.py:206-219 panel_householder; randomized.py:150-155
// _panel_rank; kernels.py:139-147 build_t_matrix).
//
// The mm x bw panel is split by rows over Q CTAs and kept in shared memory
// (global fallback when a row slab does not fit).  One grid barrier per
// column: before the barrier every CTA publishes, for the next column j, the
// partial inner products d_c = sum_{r>j} P[r,j] P[r,c] over its rows (d_j is
// the partial squared norm) and the owner of row j publishes that row; after
// the barrier every CTA reduces the Q partials in the same fixed order, so
// beta, tau and w are bit-identical in every CTA, then updates its rows
//   P[r,c] -= (tau v_r) w_c,   v_r = P[r,j] / (alpha - beta)   (kernels.py:42,52)
// and immediately forms the partials of column j+1.  The reflector convention
// is the reference's: beta = -sign(alpha)||x|| with sign(0) = +1, a nonzero
// column is always reflected, a zero column gives tau = 0.
// v is kept below the diagonal (LAPACK style) until the commit, which writes
// R (zeros below the diagonal) and the unit-lower Y only when the policy
// allows it (speculative path: all columns usable, else Status.abort).
#include "runtime.hpp"

namespace rq {

namespace {

constexpr int kPanThreads = 256;
constexpr int kMaxBw = 256;

struct PanGridArgs {
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
  unsigned int* bar;
  double* pub;    // [2][Q][2*bw]: d_c (c<bw) then row-j values (c<bw)
  double* gram;   // [Q][bw*bw] then [bw*bw] reduced
  double* gstore;
  int rpb, ldl, use_smem, cs;
};

__global__ void __launch_bounds__(kPanThreads, 1) panel_grid_kernel(PanGridArgs a) {
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int Q = gridDim.x, me = blockIdx.x;
  const int bw = a.bw, cs = a.cs, groups = kPanThreads / cs;
  const int tc = tid % cs, tg = tid / cs;
  const int64_t r0 = (int64_t)me * a.rpb;
  const int nrow = (int)imax64(0, imin64(a.mm - r0, a.rpb));
  const int ldl = a.ldl;
  double* loc = a.use_smem ? sm : a.gstore + (size_t)me * a.rpb * (size_t)bw;
  double* aux = a.use_smem ? sm + (size_t)ldl * bw : sm;
  double* part = aux;                      // [groups][bw]
  double* dsum = part + groups * bw;       // [bw]
  double* rowj = dsum + bw;                // [bw]
  double* wsh = rowj + bw;                 // [bw]
  double* taus = wsh + bw;                 // [bw]
  double* tvrow = taus + bw;               // [rpb]  tau * v_r for my rows
  double* xnext = tvrow + a.rpb;           // [rpb]  updated column j+1
  __shared__ double s_sc[4];
  __shared__ int s_usable;
  unsigned int epoch = 0;
  const int stride = 2 * bw;
  const int64_t ncols = imin64(bw, a.mm);

  // ---- load my row slab (coalesced down each column, many loads in flight)
  {
    const int total = nrow * bw;
#pragma unroll 8
    for (int e = tid; e < total; e += kPanThreads) {
      const int c = e / nrow, r = e - c * nrow;
      loc[(size_t)c * ldl + r] = a.P[(size_t)c * a.ldp + r0 + r];
    }
  }
  if (tid == 0) s_usable = (int)ncols;
  __syncthreads();

  // publish the partials of column jn over my rows r > jn (+ row jn if owned)
  auto publish = [&](int jn, const double* xc) {
    double* out = a.pub + ((size_t)(jn & 1) * Q + me) * stride;
    const int rstart = (int)imax64(0, (int64_t)jn + 1 - r0);
    for (int c = jn + tc; c < bw; c += cs) {
      const double* col = loc + (size_t)c * ldl;
      double d = 0.0;
      for (int r = rstart + tg; r < nrow; r += groups) d = __fma_rn(xc[r], col[r], d);
      part[tg * bw + c] = d;
    }
    __syncthreads();
    if (tg == 0)
      for (int c = jn + tc; c < bw; c += cs) {
        double d = part[c];
        for (int g = 1; g < groups; ++g) d = __dadd_rn(d, part[g * bw + c]);
        out[c] = d;
      }
    if (jn >= r0 && jn < r0 + nrow) {
      const int lr = (int)(jn - r0);
      for (int c = jn + tid; c < bw; c += kPanThreads) out[bw + c] = loc[(size_t)c * ldl + lr];
    }
  };

  int64_t l2 = 0, l2b = 0;
  if (ncols > 0) publish(0, loc);
  for (int j = 0; j < ncols; ++j) {
    grid_barrier(a.bar, epoch);
    const double* pb = a.pub + (size_t)(j & 1) * Q * stride;
    const int owner = (int)(j / a.rpb);
    // (1) reduce the Q partials: thread (c, g) sums its q-chunk in order,
    //     then the chunks are combined in order (identical in every CTA)
    {
      const int qlo = (int)((int64_t)tg * Q / groups), qhi = (int)((int64_t)(tg + 1) * Q / groups);
      for (int c = j + tc; c < bw; c += cs) {
        double d = 0.0;
#pragma unroll 8
        for (int q = qlo; q < qhi; ++q) d = __dadd_rn(d, pb[(size_t)q * stride + c]);
        part[tg * bw + c] = d;
        if (tg == 0) rowj[c] = pb[(size_t)owner * stride + bw + c];
      }
    }
    __syncthreads();
    if (tg == 0)
      for (int c = j + tc; c < bw; c += cs) {
        double d = part[c];
        for (int g = 1; g < groups; ++g) d = __dadd_rn(d, part[g * bw + c]);
        dsum[c] = d;
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
    // (3) w_c = v^T P[:,c] = P[j,c] + (sum_{r>j} x_r P[r,c]) / (alpha - beta);
    //     v_r = x_r / (alpha - beta) once per row (kernels.py:42), column j
    //     becomes beta on the diagonal and v below it
    for (int c = j + 1 + tid; c < bw; c += kPanThreads)
      wsh[c] = zero ? rowj[c] : __dadd_rn(rowj[c], __ddiv_rn(dsum[c], den));
    const int rj = (int)imax64(0, (int64_t)j - r0);  // first local row >= j
    {
      double* xj = loc + (size_t)j * ldl;
      for (int r = rj + tid; r < nrow; r += kPanThreads) {
        const bool diag = r0 + r == j;
        const double v = diag ? 1.0 : (zero ? xj[r] : __ddiv_rn(xj[r], den));
        tvrow[r] = __dmul_rn(tau, v);
        xj[r] = diag ? beta : v;
      }
    }
    __syncthreads();
    const bool more = j + 1 < ncols;
    // (4) updated column j+1 first (it feeds the next partials)
    if (more) {
      const double w1 = wsh[j + 1];
      double* x1 = loc + (size_t)(j + 1) * ldl;
      for (int r = rj + tid; r < nrow; r += kPanThreads) {
        const double nv = tau != 0.0 ? __dsub_rn(x1[r], __dmul_rn(tvrow[r], w1)) : x1[r];
        x1[r] = nv;
        xnext[r] = nv;
      }
    }
    __syncthreads();
    // (5) fused trailing update of columns > j+1 and the partials of step j+1
    if (more) {
      const int rs1 = (int)imax64(0, (int64_t)j + 2 - r0);  // rows > j+1
      for (int c = j + 1 + tc; c < bw; c += cs) {
        double* col = loc + (size_t)c * ldl;
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
      double* out = a.pub + ((size_t)((j + 1) & 1) * Q + me) * stride;
      if (tg == 0)
        for (int c = j + 1 + tc; c < bw; c += cs) {
          double d = part[c];
          for (int g = 1; g < groups; ++g) d = __dadd_rn(d, part[g * bw + c]);
          out[c] = d;
        }
      if (j + 1 >= r0 && j + 1 < r0 + nrow) {
        const int lr = (int)(j + 1 - r0);
        for (int c = j + 1 + tid; c < bw; c += kPanThreads) out[bw + c] = loc[(size_t)c * ldl + lr];
      }
    }
    __syncthreads();
  }

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
  if (ncommit == 0) return;  // uniform across the grid
  {
    const int total = nrow * ncommit;
#pragma unroll 4
    for (int e = tid; e < total; e += kPanThreads) {
      const int c = e / nrow, r = e - c * nrow;
      const int64_t gr = r0 + r;
      const double val = loc[(size_t)c * ldl + r];
      a.Y[(size_t)c * a.ldy + gr] = gr < c ? 0.0 : (gr == c ? 1.0 : val);
      if (gr < a.rrows) a.Rdst[(size_t)c * a.ldr + gr] = gr <= c ? val : 0.0;
    }
  }
  if (me == 0)
    for (int c = tid; c < ncommit; c += kPanThreads) a.tau[c] = taus[c];
  if (a.T == nullptr) return;

  // ---- T factor (kernels.py:139-147): G = Y^T Y (strict upper) from the
  // per-CTA partials, then T[:j,j] = -tau_j T[:j,:j] G[:j,j]
  const int nc = ncommit;
  const int npair = nc * (nc - 1) / 2;
  double* gq = a.gram + (size_t)me * npair;
  for (int e = tid; e < npair; e += kPanThreads) {
    // pair index e -> (i, j), i < j, column-major over the strict upper triangle
    int j = (int)((1.0 + sqrt(1.0 + 8.0 * e)) * 0.5);
    while (j * (j - 1) / 2 > e) --j;
    while ((j + 1) * j / 2 <= e) ++j;
    const int i = e - j * (j - 1) / 2;
    const int rs = (int)imax64(0, (int64_t)j - r0);  // rows >= j carry both
    const double* yi = loc + (size_t)i * ldl;
    const double* yj = loc + (size_t)j * ldl;
    double g = 0.0;
    for (int r = rs; r < nrow; ++r) {
      const double vj = (r0 + r == j) ? 1.0 : yj[r];
      g = __fma_rn(yi[r], vj, g);
    }
    gq[e] = g;
  }
  grid_barrier(a.bar, epoch);
  double* gfin = a.gram + (size_t)Q * npair;
  {
    const int per = (npair + Q - 1) / Q;
    const int lo = me * per, hi = min(npair, lo + per);
    for (int e = lo + tid; e < hi; e += kPanThreads) {
      double g = 0.0;
#pragma unroll 8
      for (int q = 0; q < Q; ++q) g = __dadd_rn(g, a.gram[(size_t)q * npair + e]);
      gfin[e] = g;
    }
  }
  grid_barrier(a.bar, epoch);
  if (me != 0) return;
  const bool tsm = a.use_smem && ldl >= nc;
  double* Tw = tsm ? loc : a.T;          // T workspace, column-major
  const int ldtw = tsm ? ldl : (int)a.ldt;
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

void panel_qr_grid(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
              const PanelOut& out, double tol, PanelPolicy policy, bool raise_abort, Status* st,
              int64_t i0, cudaStream_t s) {
  if (bw < 1 || bw > kMaxBw) throw InvalidArg("panel width must be in [1, 256]");
  if (mm < 1) throw InvalidArg("panel needs at least one row");
  int Q = (int)std::min<int64_t>(h.num_sms, (mm + 127) / 128);
  Q = std::max(Q, 1);
  const int rpb = (int)((mm + Q - 1) / Q);
  Q = (int)((mm + rpb - 1) / rpb);
  int cs = 1;
  while (cs < bw && cs < kPanThreads) cs <<= 1;
  const int groups = kPanThreads / cs;
  const int ldl = rpb | 1;
  const size_t aux = ((size_t)groups * bw + 5 * (size_t)bw + 2 * (size_t)rpb + 8) * 8;
  const size_t store = (size_t)ldl * bw * 8;
  const bool use_smem = store + aux <= h.smem_optin - 2048;
  const size_t smem = (use_smem ? store : 0) + aux;
  PanGridArgs a{};
  a.mm = mm; a.bw = (int)bw; a.P = P; a.ldp = ldp;
  a.Rdst = out.Rdst; a.ldr = out.ldr; a.rrows = out.rrows;
  a.Y = out.Y; a.ldy = out.ldy; a.tau = out.tau; a.T = out.T; a.ldt = out.ldt;
  a.tol = tol; a.policy = (int)policy; a.raise_abort = raise_abort ? 1 : 0; a.i0 = i0;
  a.st = st;
  a.bar = (unsigned int*)h.buf("pang_bar", 64, s);
  a.pub = (double*)h.buf("pang_pub", (size_t)2 * Q * 2 * bw * 8, s);
  a.gram = out.T ? (double*)h.buf("pang_gram", (size_t)(Q + 1) * bw * bw * 4 + 64, s) : nullptr;
  a.gstore = use_smem ? nullptr : (double*)h.buf("pang_gstore", (size_t)Q * rpb * bw * 8, s);
  a.rpb = rpb; a.ldl = use_smem ? ldl : rpb; a.use_smem = use_smem ? 1 : 0; a.cs = cs;
  RQ_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
  static size_t attr = 0;
  if (smem > attr) {
    RQ_CUDA(cudaFuncSetAttribute(panel_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 48 * 1024)));
    attr = std::max<size_t>(smem, 48 * 1024);
  }
  void* args[] = {&a};
  ProfScope prof(h, kProfPanel, 2.0 * mm * bw * bw, 16.0 * mm * bw, s);
  count_launch();
  RQ_CUDA(cudaLaunchCooperativeKernel((void*)panel_grid_kernel, dim3(Q), dim3(kPanThreads), args,
                                      smem, s));
}

}  // namespace rq
