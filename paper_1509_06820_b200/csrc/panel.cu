// K5: panel Householder QR + _panel_rank (qrcp.py:206-219 panel_householder;
// randomized.py:150-155 _panel_rank).  The T factor (kernels.py:139-147) is
// built afterwards by t_factor() from a DMMA Gram GEMM.
//
// The mm x bw panel is split by rows over Q CTAs; every thread OWNS whole
// rows (row-major shared-memory slab, odd leading dimension, rows past the
// budget spill to L2), so one pass per column both applies the reflector and
// forms the next column's partial inner products without any cross-thread
// hand-off:
//   P[r,c] -= (tau v_r) w_c,   v_r = P[r,j] / (alpha - beta)   (kernels.py:42,52)
//   d_c    += P'[r,j+1] P'[r,c]      (r > j+1)
// The partial vectors are reduced within a warp by a 31-shuffle transpose
// reduction, across warps in shared memory, and across CTAs by the exchange:
// either one thread-block cluster (Q <= 16, DSMEM + cluster barrier ~0.23 us)
// or a cooperative grid (Q <= 64, L2 buffers + grid barrier ~1.2 us).  Every
// CTA reduces the Q partials in the same fixed order, so alpha, beta, tau and
// w are bit-identical everywhere.  Per column: one exchange + two block
// barriers.  Reflector convention is the reference's: beta = -sign(alpha)||x||,
// sign(0) = +1, a nonzero column is always reflected, a zero column gives
// tau = 0.  v is kept below the diagonal until the commit, which writes R
// (zeros below the diagonal) and unit-lower Y only when the policy allows it
// (speculative path: all columns usable, else Status.abort).
#include <cooperative_groups.h>

#include "runtime.hpp"

namespace cg = cooperative_groups;

namespace rq {

namespace {

constexpr int kPanThreads = 256;
constexpr int kMaxBw = 256;
constexpr int kMaxCluster = 16;
constexpr int kMaxGrid = 64;
constexpr int kRowsPerThread = 4;   // rpb <= 1024
constexpr int kChunk = 32;          // columns per register chunk

struct PanArgs {
  int64_t mm;
  int bw;
  const double* P; int64_t ldp;
  double* Rdst; int64_t ldr; int64_t rrows;
  double* Y; int64_t ldy;
  double* tau;
  double tol;
  int policy;
  int raise_abort;
  int64_t i0;
  Status* st;
  double* gstore;          // spill rows [Q][rpb - nrs][ldl]
  int rpb, ldl, nrs;       // rows per CTA, row stride (odd), rows kept in smem
  // grid exchange
  unsigned int* bar;
  double* gpub;            // [2][Q][2*bw]
  long long* dbg;          // optional phase timers (CTA 0, thread 0)
  const int* skip;         // panel_fast verdict: nonzero = already committed
};

// 32 per-lane values -> lane l holds the warp sum of column l (31 shuffles,
// fixed combination order)
RQ_DEV double warp_transpose_sum(double (&d)[kChunk]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double keep = up ? d[i + off] : d[i];
      const double give = up ? d[i] : d[i + off];
      const double got = __shfl_xor_sync(0xffffffffu, give, off);
      d[i] = up ? __dadd_rn(got, keep) : __dadd_rn(keep, got);
    }
  }
  return d[0];
}

template <bool kCluster>
__global__ void __launch_bounds__(kPanThreads, 1) panel_kernel(PanArgs a) {
  if (aborted(a.st)) return;
  if (a.skip != nullptr && *(volatile const int*)a.skip != 0) return;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kPanThreads / 32;
  int Q, me;
  if constexpr (kCluster) {
    Q = (int)cg::this_cluster().num_blocks();
    me = (int)cg::this_cluster().block_rank();
  } else {
    Q = gridDim.x;
    me = blockIdx.x;
  }
  const int bw = a.bw, ldl = a.ldl, nrs = a.nrs;
  const int64_t r0 = (int64_t)me * a.rpb;
  const int nrow = (int)imax64(0, imin64(a.mm - r0, a.rpb));
  double* gsp = a.gstore ? a.gstore + (size_t)me * (a.rpb - nrs) * ldl : nullptr;
  auto rowp = [&](int r) -> double* {
    return r < nrs ? sm + (size_t)r * ldl : gsp + (size_t)(r - nrs) * ldl;
  };
  double* aux = sm + (size_t)nrs * ldl;
  double* xpub = aux;                  // [2][2*bw] partials + owner row (cluster exchange)
  double* wpart = xpub + 4 * bw;       // [NW][bw] per-warp partial sums
  double* dsum = wpart + NW * bw;      // [bw]
  double* rowj = dsum + bw;            // [bw]
  double* taus = rowj + bw;            // [bw]
  double* wsh = taus + bw;             // [bw] w of the current step
  __shared__ int s_usable;
  unsigned int epoch = 0;
  const int stride = 2 * bw;
  const int64_t ncols = imin64(bw, a.mm);
  auto xsync = [&]() {
    if constexpr (kCluster) cg::this_cluster().sync();
    else grid_barrier(a.bar, epoch);
  };
  auto pub_out = [&](int par) -> double* {
    if constexpr (kCluster) return xpub + (size_t)par * stride;
    else return a.gpub + ((size_t)par * Q + me) * stride;
  };

  // ---- load my rows (coalesced down each global column)
  {
    const int total = nrow * bw;
#pragma unroll 8
    for (int e = tid; e < total; e += kPanThreads) {
      const int c = e / nrow, r = e - c * nrow;
      rowp(r)[c] = a.P[(size_t)c * a.ldp + r0 + r];
    }
  }
  if (tid == 0) s_usable = (int)ncols;
  __syncthreads();

  // partial vector for column jn (rows > jn): per-thread registers, warp
  // transpose-reduce, per-warp slots, then the block sum and the owner row
  auto finish_partials = [&](int jn) {
    __syncthreads();
    double* out = pub_out(jn & 1);
    for (int c = jn + tid; c < bw; c += kPanThreads) {
      double d = wpart[c];
      for (int w = 1; w < NW; ++w) d = __dadd_rn(d, wpart[w * bw + c]);
      out[c] = d;
    }
    if (jn >= r0 && jn < r0 + nrow) {
      const double* rr = rowp((int)(jn - r0));
      for (int c = jn + tid; c < bw; c += kPanThreads) out[bw + c] = rr[c];
    }
  };

  // initial partials of column 0
  for (int cb = 0; cb < bw; cb += kChunk) {
    double d[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) d[i] = 0.0;
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      const int r = tid + k * kPanThreads;
      if (r < nrow && r0 + r > 0) {
        const double* rr = rowp(r);
        const double x = rr[0];
#pragma unroll
        for (int i = 0; i < kChunk; ++i)
          if (cb + i < bw) d[i] = __fma_rn(x, rr[cb + i], d[i]);
      }
    }
    const double s = warp_transpose_sum(d);
    if (cb + lane < bw) wpart[warp * bw + cb + lane] = s;
  }
  finish_partials(0);

  int64_t l2 = 0, l2b = 0;
  long long tm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  const bool timing = a.dbg != nullptr && me == 0 && tid == 0;
  auto mark = [&](int k) {
    if (timing) {
      const long long t = clock64();
      tm[k] += t - tlast;
      tlast = t;
    }
  };
  for (int j = 0; j < ncols; ++j) {
    mark(5);
    xsync();
    mark(0);
    const int par = j & 1;
    const int owner = (int)(j / a.rpb);
    // (A) fixed-order reduction of the Q partial vectors
    for (int c = j + tid; c < bw; c += kPanThreads) {
      double d = 0.0;
      if constexpr (kCluster) {
        double v[kMaxCluster];
#pragma unroll
        for (int q = 0; q < kMaxCluster; ++q)
          if (q < Q) v[q] = cg::this_cluster().map_shared_rank(xpub, q)[par * stride + c];
#pragma unroll
        for (int q = 0; q < kMaxCluster; ++q)
          if (q < Q) d = __dadd_rn(d, v[q]);
        rowj[c] = cg::this_cluster().map_shared_rank(xpub, owner)[par * stride + bw + c];
      } else {
        const double* g = a.gpub + (size_t)par * Q * stride + c;
        double v[kMaxGrid];
#pragma unroll
        for (int q = 0; q < kMaxGrid; ++q)
          if (q < Q) v[q] = g[(size_t)q * stride];
#pragma unroll
        for (int q = 0; q < kMaxGrid; ++q)
          if (q < Q) d = __dadd_rn(d, v[q]);
        rowj[c] = a.gpub[((size_t)par * Q + owner) * stride + bw + c];
      }
      dsum[c] = d;
    }
    __syncthreads();
    mark(1);
    // (B) reflector scalars (kernels.py:35-44), computed redundantly by every thread
    const double alpha = rowj[j];
    const double norm = sqrt(__fma_rn(alpha, alpha, dsum[j]));
    double beta = 0.0, tau = 0.0, den = 1.0;
    const bool zero = norm == 0.0;
    if (!zero) {
      beta = alpha >= 0.0 ? -norm : norm;
      den = __dsub_rn(alpha, beta);
      tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
    }
    const double rinv = zero ? 0.0 : 1.0 / den;
    // w_c = P[j,c] + (sum_{r>j} x_r P[r,c]) / (alpha - beta), once per column
    for (int c = j + 1 + tid; c < bw; c += kPanThreads) wsh[c] = __fma_rn(dsum[c], rinv, rowj[c]);
    if (tid == 0) {
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
    const bool more = j + 1 < ncols;
    // (C) one pass over my rows: v, update of columns > j (w_c = P[j,c] +
    //     (sum_{r>j} x_r P[r,c]) / (alpha - beta)), partials of column j+1
    double tvr[kRowsPerThread];
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      const int r = tid + k * kPanThreads;
      tvr[k] = 0.0;
      if (r < nrow && r0 + r >= j) {
        double* rr = rowp(r);
        const bool diag = r0 + r == j;
        const double v = diag ? 1.0 : (zero ? rr[j] : __dmul_rn(rr[j], rinv));
        tvr[k] = __dmul_rn(tau, v);
        rr[j] = diag ? beta : v;
      }
    }
    mark(2);
    if (!more) break;
    __syncthreads();  // wsh complete
    const double w1 = wsh[j + 1];
    // updated x' = P'[r, j+1] of my rows, before any chunk rewrites column j+1
    double x1r[kRowsPerThread];
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      const int r = tid + k * kPanThreads;
      x1r[k] = 0.0;
      if (r < nrow && r0 + r >= j) {
        const double old = rowp(r)[j + 1];
        x1r[k] = tau != 0.0 ? __dsub_rn(old, __dmul_rn(tvr[k], w1)) : old;
      }
    }
    for (int cb = j + 1; cb < bw; cb += kChunk) {
      double d[kChunk];
#pragma unroll
      for (int i = 0; i < kChunk; ++i) d[i] = 0.0;
#pragma unroll
      for (int k = 0; k < kRowsPerThread; ++k) {
        const int r = tid + k * kPanThreads;
        if (r < nrow && r0 + r >= j) {
          double* rr = rowp(r);
          const double tv = tvr[k];
          const double x1 = x1r[k];
          const bool below = r0 + r > j + 1;
#pragma unroll
          for (int i = 0; i < kChunk; ++i) {
            const int c = cb + i;
            if (c < bw) {
              double nv = rr[c];
              if (tau != 0.0) nv = __dsub_rn(nv, __dmul_rn(tv, wsh[c]));
              rr[c] = nv;
              if (below) d[i] = __fma_rn(x1, nv, d[i]);
            }
          }
        }
      }
      const double s = warp_transpose_sum(d);
      if (cb + lane < bw) wpart[warp * bw + cb + lane] = s;
    }
    mark(3);
    finish_partials(j + 1);
    mark(4);
  }
  if (timing) {
    for (int k = 0; k < 6; ++k) a.dbg[k] = tm[k];
    a.dbg[7] = ncols;
  }
  xsync();  // every CTA is done reading the others' partials

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
  if (ncommit > 0) {
    const int total = nrow * ncommit;
#pragma unroll 4
    for (int e = tid; e < total; e += kPanThreads) {
      const int c = e / nrow, r = e - c * nrow;
      const int64_t gr = r0 + r;
      const double val = rowp(r)[c];
      a.Y[(size_t)c * a.ldy + gr] = gr < c ? 0.0 : (gr == c ? 1.0 : val);
      if (gr < a.rrows) a.Rdst[(size_t)c * a.ldr + gr] = gr <= c ? val : 0.0;
    }
    if (me == 0)
      for (int c = tid; c < ncommit; c += kPanThreads) a.tau[c] = taus[c];
  }
  if constexpr (kCluster) cg::this_cluster().sync();  // peers' DSMEM reads are done
}

}  // namespace

void panel_qr(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
              const PanelOut& out, double tol, PanelPolicy policy, bool raise_abort, Status* st,
              int64_t i0, cudaStream_t s, bool allow_fast, bool fast_aborts) {
  if (bw < 1 || bw > kMaxBw) throw InvalidArg("panel width must be in [1, 256]");
  if (mm < 1) throw InvalidArg("panel needs at least one row");
  const bool grid = h.force_panel == 1 || (h.force_panel == 0 && mm > h.panel_cluster_max_rows);
  int Q = 1;
  if (grid) {
    Q = (int)std::min<int64_t>(kMaxGrid, (mm + 127) / 128);
    Q = std::max(Q, 1);
  } else {
    while (Q < kMaxCluster && (int64_t)Q * h.panel_rows_per_cta < mm) Q <<= 1;
  }
  const int rpb = (int)((mm + Q - 1) / Q);
  if (rpb > kRowsPerThread * kPanThreads) throw InvalidArg("panel too tall for the kernel");
  const int ldl = (int)(bw | 1);
  const size_t aux = ((size_t)4 * bw + (size_t)(kPanThreads / 32) * bw + 4 * (size_t)bw + 8) * 8;
  if (aux > h.smem_optin - 4096) throw InvalidArg("panel too wide for shared memory");
  // CholeskyQR2 + reconstruction first (panel_fast.cu); this kernel then
  // only runs when that path declined the panel
  const bool decline_aborts = raise_abort && fast_aborts;
  const int* skip =
      allow_fast ? panel_fast(h, mm, bw, P, ldp, out, tol, st, s, decline_aborts, i0) : nullptr;
  if (skip != nullptr && decline_aborts) return;   // speculative: a decline rewinds the block
  const size_t rowbytes = (size_t)ldl * 8;
  const int nrs = (int)std::min<size_t>(rpb, (h.smem_optin - 4096 - aux) / rowbytes);
  const size_t smem = (size_t)nrs * rowbytes + aux;
  PanArgs a{};
  a.mm = mm; a.bw = (int)bw; a.P = P; a.ldp = ldp;
  a.Rdst = out.Rdst; a.ldr = out.ldr; a.rrows = out.rrows;
  a.Y = out.Y; a.ldy = out.ldy; a.tau = out.tau;
  a.tol = tol; a.policy = (int)policy; a.raise_abort = raise_abort ? 1 : 0; a.i0 = i0;
  a.st = st;
  a.gstore = nrs < rpb ? (double*)h.buf("pan_gstore", (size_t)Q * (rpb - nrs) * rowbytes, s)
                       : nullptr;
  a.rpb = rpb; a.ldl = ldl; a.nrs = nrs;
  a.dbg = h.dbg;
  a.skip = skip;
  {
    ProfScope prof(h, kProfPanel, 2.0 * mm * bw * bw, 16.0 * mm * bw, s);
    count_launch();
    if (grid) {
      a.bar = (unsigned int*)h.buf("pan_bar", 64, s);
      a.gpub = (double*)h.buf("pan_gpub", (size_t)2 * Q * 2 * bw * 8, s);
      RQ_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
      kernel_attr((const void*)panel_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                  (int)std::max<size_t>(smem, 48 * 1024));
      void* args[] = {&a};
      RQ_CUDA(cudaLaunchCooperativeKernel((void*)panel_kernel<false>, dim3(Q), dim3(kPanThreads),
                                          args, smem, s));
    } else {
      kernel_attr((const void*)panel_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      kernel_attr((const void*)panel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                  (int)std::max<size_t>(smem, 48 * 1024));
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
      RQ_CUDA(cudaLaunchKernelEx(&cfg, panel_kernel<true>, a));
    }
  }
  if (out.T != nullptr) {
    // T factor of the committed columns (kernels.py:139-147); after a failed
    // speculative commit the Status predicate turns this into a no-op
    // (already written by the fast path when it committed: its flag word
    // doubles as the Status predicate of these launches)
    t_factor(h, out.Y, out.ldy, mm, bw, out.tau, out.T, out.ldt, s,
             skip != nullptr ? (const Status*)skip : st);
  }
}

}  // namespace rq
