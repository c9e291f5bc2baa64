// K5: panel Householder QR + _panel_rank + T factor, one persistent
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
  unsigned int* bar;
  double* pub;    // [2][Q][2*bw]: d_c (c<bw) then row-j values (c<bw)
  double* gram;   // [Q][bw*bw] then [bw*bw] reduced
  double* gstore;
  int rpb, ldl, use_smem, cs;
};

__global__ void __launch_bounds__(kPanThreads, 1) panel_kernel(PanArgs a) {
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
  double* betas = taus + bw;               // [bw]
  __shared__ double s_sc[4];
  __shared__ int s_usable;
  unsigned int epoch = 0;
  const int stride = 2 * bw;

  // load my row slab (column-major, ld = ldl)
  for (int c = 0; c < bw; ++c)
    for (int r = tid; r < nrow; r += kPanThreads)
      loc[(size_t)c * ldl + r] = a.P[(size_t)c * a.ldp + r0 + r];
  if (tid == 0) s_usable = bw;
  __syncthreads();

  // partials of column jn over my rows r > jn, plus row jn if I own it
  auto publish = [&](int jn) {
    const int par = jn & 1;
    double* out = a.pub + ((size_t)par * Q + me) * stride;
    const double* xcol = loc + (size_t)jn * ldl;
    const int rstart = (int)imax64(0, (int64_t)jn + 1 - r0);
    for (int c = jn + tc; c < bw; c += cs) {
      const double* col = loc + (size_t)c * ldl;
      double d = 0.0;
      for (int r = rstart + tg; r < nrow; r += groups) d = __fma_rn(xcol[r], col[r], d);
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
    __syncthreads();
  };

  const int64_t ncols = imin64(bw, a.mm);
  int64_t l2 = 0, l2b = 0;
  if (ncols > 0) publish(0);
  for (int j = 0; j < ncols; ++j) {
    grid_barrier(a.bar, epoch);
    const int par = j & 1;
    const int owner = (int)(j / a.rpb);
    // reduce partials in fixed q order (identical in every CTA)
    for (int c = j + tid; c < bw; c += kPanThreads) {
      double d = 0.0;
      for (int q = 0; q < Q; ++q) d = __dadd_rn(d, a.pub[((size_t)par * Q + q) * stride + c]);
      dsum[c] = d;
      rowj[c] = a.pub[((size_t)par * Q + owner) * stride + bw + c];
    }
    __syncthreads();
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
      betas[j] = beta;
      if (s_usable == bw && fabs(beta) <= a.tol) s_usable = j;  // _panel_rank
      if (me == 0) {
        const int64_t cols = bw - j - 1;
        if (tau != 0.0 && cols > 0) {
          l2 += 4 * (a.mm - j) * cols;
          l2b += 16 * (a.mm - j) * cols;
        }
      }
    }
    __syncthreads();
    const double tau = s_sc[1], den = s_sc[2];
    const bool zero = s_sc[3] == 0.0;
    // w_c = v^T P[:,c] = P[j,c] + (sum_{r>j} x_r P[r,c]) / (alpha - beta)
    for (int c = j + 1 + tid; c < bw; c += kPanThreads)
      wsh[c] = zero ? rowj[c] : __dadd_rn(rowj[c], __ddiv_rn(dsum[c], den));
    __syncthreads();
    const double* xcol = loc + (size_t)j * ldl;
    const int rj = (int)imax64(0, (int64_t)j - r0);  // first local row >= j
    if (tau != 0.0) {
      for (int c = j + 1 + tc; c < bw; c += cs) {
        double* col = loc + (size_t)c * ldl;
        const double w = wsh[c];
        for (int r = rj + tg; r < nrow; r += groups) {
          const int64_t gr = r0 + r;
          const double v = (gr == j) ? 1.0 : __ddiv_rn(xcol[r], den);
          col[r] = __dsub_rn(col[r], __dmul_rn(__dmul_rn(tau, v), w));
        }
      }
    }
    __syncthreads();
    // column j: beta on the diagonal, v below it (scaled reflector)
    for (int r = rj + tid; r < nrow; r += kPanThreads) {
      const int64_t gr = r0 + r;
      double* x = loc + (size_t)j * ldl + r;
      if (gr == j) *x = s_sc[0];
      else if (!zero) *x = __ddiv_rn(*x, den);
    }
    __syncthreads();
    if (j + 1 < ncols) publish(j + 1);
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
  for (int c = 0; c < ncommit; ++c) {
    for (int r = tid; r < nrow; r += kPanThreads) {
      const int64_t gr = r0 + r;
      const double val = loc[(size_t)c * ldl + r];
      a.Y[(size_t)c * a.ldy + gr] = gr < c ? 0.0 : (gr == c ? 1.0 : val);
      if (gr < a.rrows) a.Rdst[(size_t)c * a.ldr + gr] = gr <= c ? val : 0.0;
    }
  }
  if (me == 0)
    for (int c = tid; c < ncommit; c += kPanThreads) a.tau[c] = taus[c];
  if (a.T == nullptr) return;

  // ---- T factor (kernels.py:139-147): G = Y^T Y (strict upper), then the
  // forward column recurrence T[:j,j] = -tau_j T[:j,:j] G[:j,j]
  const int nc = ncommit;
  double* gq = a.gram + (size_t)me * bw * bw;
  for (int e = tid; e < nc * nc; e += kPanThreads) {
    const int i = e % nc, j = e / nc;
    if (i >= j) continue;
    double g = 0.0;
    const int rs = (int)imax64(0, (int64_t)j - r0);  // rows >= j carry both
    for (int r = rs; r < nrow; ++r) {
      const int64_t gr = r0 + r;
      const double yi = gr == i ? 1.0 : loc[(size_t)i * ldl + r];
      const double yj = gr == j ? 1.0 : loc[(size_t)j * ldl + r];
      g = __fma_rn(yi, yj, g);
    }
    gq[i + (size_t)j * bw] = g;
  }
  grid_barrier(a.bar, epoch);
  double* gfin = a.gram + (size_t)Q * bw * bw;
  {
    const int total = nc * nc;
    const int per = (total + Q - 1) / Q;
    for (int e = me * per + tid; e < min(total, (me + 1) * per); e += kPanThreads) {
      const int i = e % nc, j = e / nc;
      if (i >= j) continue;
      double g = 0.0;
      for (int q = 0; q < Q; ++q) g = __dadd_rn(g, a.gram[(size_t)q * bw * bw + i + (size_t)j * bw]);
      gfin[i + (size_t)j * bw] = g;
    }
  }
  grid_barrier(a.bar, epoch);
  if (me != 0) return;
  double* Tsh = part;  // reuse: [bw*bw] would not fit for big bw; write T directly
  (void)Tsh;
  for (int j = 0; j < nc; ++j) {
    // T[:j, j] = -tau_j * (T[:j,:j] @ g), g = G[:j, j]
    for (int i = tid; i < j; i += kPanThreads) {
      double t = 0.0;
      for (int l = i; l < j; ++l)
        t = __fma_rn(a.T[i + (size_t)l * a.ldt], gfin[l + (size_t)j * bw], t);
      wsh[i] = t;
    }
    __syncthreads();
    for (int i = tid; i < nc; i += kPanThreads) {
      double v;
      if (i < j) v = __dmul_rn(-taus[j], wsh[i]);
      else if (i == j) v = taus[j];
      else v = 0.0;
      a.T[i + (size_t)j * a.ldt] = v;
    }
    __syncthreads();
  }
}

}  // namespace

void panel_qr(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
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
  const size_t aux = ((size_t)groups * bw + 5 * (size_t)bw + 8) * 8;
  const size_t store = (size_t)ldl * bw * 8;
  const bool use_smem = store + aux <= h.smem_optin - 2048;
  const size_t smem = (use_smem ? store : 0) + aux;
  PanArgs a{};
  a.mm = mm; a.bw = (int)bw; a.P = P; a.ldp = ldp;
  a.Rdst = out.Rdst; a.ldr = out.ldr; a.rrows = out.rrows;
  a.Y = out.Y; a.ldy = out.ldy; a.tau = out.tau; a.T = out.T; a.ldt = out.ldt;
  a.tol = tol; a.policy = (int)policy; a.raise_abort = raise_abort ? 1 : 0; a.i0 = i0;
  a.st = st;
  a.bar = (unsigned int*)h.buf("pan_bar", 64, s);
  a.pub = (double*)h.buf("pan_pub", (size_t)2 * Q * 2 * bw * 8, s);
  a.gram = out.T ? (double*)h.buf("pan_gram", (size_t)(Q + 1) * bw * bw * 8, s) : nullptr;
  a.gstore = use_smem ? nullptr : (double*)h.buf("pan_gstore", (size_t)Q * rpb * bw * 8, s);
  a.rpb = rpb; a.ldl = use_smem ? ldl : rpb; a.use_smem = use_smem ? 1 : 0; a.cs = cs;
  RQ_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
  static size_t attr = 0;
  if (smem > attr) {
    RQ_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(smem, 48 * 1024)));
    attr = std::max<size_t>(smem, 48 * 1024);
  }
  void* args[] = {&a};
  ProfScope prof(h, kProfPanel, 2.0 * mm * bw * bw, 16.0 * mm * bw, s);
  count_launch();
  RQ_CUDA(cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(Q), dim3(kPanThreads), args,
                                      smem, s));
}

}  // namespace rq
