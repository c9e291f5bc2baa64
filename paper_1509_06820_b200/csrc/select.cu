// K4: pivot-block selection = `want` greedy steps of column-pivoted
// Householder QR on the small (b+p) x nt Gaussian sample, in one persistent
// kernel (randomized.py:85-104 -> qrcp.py:63-84, NormTracker
// kernels.py:196-233, form/apply_reflector kernels.py:26-56).
//
// Layout: the sample's columns are dealt out to P CTAs in contiguous chunks,
// one column per thread, resident in shared memory (columns past the budget
// spill to global/L2).  Columns never move: a swap only relabels logical
// positions.  One step costs one exchange + one block barrier:
//   exchange: every CTA publishes its local best (norm, position) and that
//     column; then either a cluster barrier with DSMEM reads (P <= 16 CTAs of
//     one thread-block cluster, small samples) or a grid barrier with
//     L2-resident buffers (all SMs, wide samples)
//   every WARP then redundantly reduces the P candidates (total order:
//     larger norm, then lower position = np.argmax first-max), fetches the
//     pivot column and forms the reflector -- identical bits everywhere, no
//     block barrier needed
//   every thread applies H_j to its own column, downdates its norm with the
//     sqrt(eps) recompute guard, and the block argmax publishes the next
//     candidate.
// Initial norms use numpy's pairwise summation, so they are bit-identical to
// np.linalg.norm(B, axis=0).
#include <cooperative_groups.h>

#include "runtime.hpp"

namespace cg = cooperative_groups;

namespace rq {

namespace {

constexpr int kSelThreads = 512;
constexpr int kMaxCluster = 16;

struct SelArgs {
  int ell, nt, want;
  int pbits;        // position bits of the argmax key: 16, or 20 for samples wider than 65535 columns
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
  // grid exchange (global/L2)
  unsigned int* bar;
  unsigned long long* gkey;  // [3] rotating candidate keys
  // fused exchange (v5 grid variant): {arrival count, max key} pairs read with
  // one 16-byte acquire load, so the barrier's last poll also delivers the key
  ulonglong2* pair;          // [3], rotating with the step like gkey (nullptr: off)
  double* gcol;     // [2][P][ell+1]
  double* gsq;      // [P]
  long long* dbg;   // optional phase timers (CTA 0, thread 0): [8] cycles
};

RQ_DEV double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// Packed argmax key: the top 48 bits of the (non-negative) norm's IEEE
// pattern, then the complemented 16-bit logical position (ties -> lowest
// position, np.argmax first-max).  Unsigned order of keys = reference order
// of candidates up to a 2^-36 relative norm resolution (a near-tie far inside
// the downdating error).  0 = no candidate.  The owner CTA of a position is
// read from a position -> owner map every CTA keeps identically.  Samples
// wider than 65535 columns take 20 position bits (44 norm bits, a 2^-32 band).
RQ_DEV unsigned long long make_key(double nrm, int pos, int pb) {
  const unsigned long long hi = ((unsigned long long)__double_as_longlong(nrm)) >> pb;
  return (hi << pb) | (unsigned long long)(((1 << pb) - 1) - pos);
}
RQ_DEV int key_pos(unsigned long long k, int pb) {
  const int mask = (1 << pb) - 1;
  return mask - (int)(k & (unsigned long long)mask);
}

template <bool kCluster>
__global__ void __launch_bounds__(kSelThreads, 1) select_kernel(SelArgs a) {
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSelThreads / 32;
  constexpr int NG = kSelThreads / 8;          // 8-lane column groups
  const int grp = tid >> 3, gl = tid & 7;
  const unsigned gmask = 0xffu << (lane & 24);  // my group's lanes
  int P, me;
  if constexpr (kCluster) {
    P = (int)cg::this_cluster().num_blocks();
    me = (int)cg::this_cluster().block_rank();
  } else {
    P = gridDim.x;
    me = blockIdx.x;
  }
  const int ell = a.ell, ldl = a.ldl, ncs = a.ncs;
  const int pb = a.pbits;
  const int c0 = me * a.cpb;
  const int ncol = max(0, min(a.nt - c0, a.cpb));
  double* gsp = a.gstore ? a.gstore + (size_t)me * (a.cpb - ncs) * ldl : nullptr;
  auto colp = [&](int c) -> double* {
    return c < ncs ? sm + (size_t)c * ldl : gsp + (size_t)(c - ncs) * ldl;
  };
  const int cstride = ell + 1;               // published column + its exact norm
  double* meta = sm + (size_t)ncs * ldl;
  double* vbuf = meta;                       // [ell] v
  double* tvbuf = vbuf + ell;                // [ell] tau*v
  double* ccol = tvbuf + ell;                // [2][ell+1] my published candidate (cluster)
  double* nrm = ccol + 2 * cstride;          // [cpb]
  double* orig = nrm + a.cpb;                // [cpb]
  int* pos = (int*)(orig + a.cpb);           // [cpb]
  unsigned char* omap = (unsigned char*)(pos + a.cpb);  // [nt] position -> owner CTA
  __shared__ unsigned long long s_key[3][kMaxCluster];  // pushed candidate keys [slot][src]
  __shared__ unsigned long long s_bkey;      // block best key
  __shared__ double s_sq[kMaxCluster];
  __shared__ double s_all[160];
  __shared__ double s_step[2];
  __shared__ int s_stepi[2];
  unsigned int epoch = 0;

  auto xsync = [&]() {
    if constexpr (kCluster) cg::this_cluster().sync();
    else grid_barrier(a.bar, epoch);
  };
  // cluster-wide best key of a slot: max over the per-source entries (cluster)
  // or the global atomic max (grid); warp 0 only
  auto slot_max = [&](int slot) -> unsigned long long {
    unsigned long long k = 0ull;
    if constexpr (kCluster) {
      if (lane < P) k = s_key[slot][lane];
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
        k = o > k ? o : k;
      }
    } else {
      k = __ldcg(a.gkey + slot);
    }
    return k;
  };

  // ---- load my columns; initial norms (pairwise, bit-identical to numpy)
  {
    const int total = ncol * ell;
#pragma unroll 4
    for (int e = tid; e < total; e += kSelThreads) {
      const int c = e / ell, i = e - c * ell;
      colp(c)[i] = a.B[(size_t)(c0 + c) * a.ldb + i];
    }
  }
  for (int e = tid; e < 3 * kMaxCluster; e += kSelThreads) (&s_key[0][0])[e] = 0ull;
  for (int q = tid; q < a.nt; q += kSelThreads) omap[q] = (unsigned char)(q / a.cpb);
  if (!kCluster && me == 0 && tid < 3) a.gkey[tid] = 0ull;
  __syncthreads();
  double mysq = 0.0;
  for (int c = tid; c < ncol; c += kSelThreads) {
    const double sq = pairwise_sumsq(colp(c), ell, 1);
    const double nv = sqrt(sq);
    nrm[c] = nv;
    orig[c] = __dmul_rn(nv, nv);
    pos[c] = c0 + c;
    mysq = __dadd_rn(mysq, sq);
  }
  {
    const double v = warp_sum(mysq);
    if (lane == 0) s_all[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t = __dadd_rn(t, s_all[w]);
      s_bkey = 0ull;
      if constexpr (kCluster) {
        for (int q = 0; q < P; ++q) cg::this_cluster().map_shared_rank(s_sq, q)[me] = t;
      } else {
        a.gsq[me] = t;
      }
    }
  }
  xsync();  // key slots are zero everywhere before anyone publishes

  // publish my block's best candidate (group leaders already atomically
  // maxed their keys into s_bkey) into key slot `slot`, column parity `par`
  auto publish = [&](int slot, int par) {
    __syncthreads();
    const unsigned long long bk = s_bkey;
    if (bk != 0ull) {
      if constexpr (kCluster) {
        if (tid < P) cg::this_cluster().map_shared_rank(&s_key[slot][0], tid)[me] = bk;
      } else {
        if (tid == 0) atomicMax(a.gkey + slot, bk);
      }
      // the winning group copies its column (+ exact norm) to the publish slot
      const int bpos = key_pos(bk, pb);
      for (int c = grp; c < ncol; c += NG) {
        if (pos[c] != bpos) continue;
        const double* src = colp(c);
        double* dst = kCluster ? ccol + par * cstride : a.gcol + ((size_t)par * P + me) * cstride;
        for (int i = gl; i < ell; i += 8) dst[i] = src[i];
        if (gl == 0) dst[ell] = nrm[c];
      }
    }
  };

  // step-0 candidates
  for (int c = grp; c < ncol; c += NG)
    if (gl == 0) atomicMax(&s_bkey, make_key(nrm[c], pos[c], pb));
  publish(0, 0);
  xsync();
  double tol;
  {
    for (int q = tid; q < P; q += kSelThreads) {
      if constexpr (kCluster) s_all[q] = s_sq[q];
      else s_all[q] = a.gsq[q];
    }
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < P; ++q) t = __dadd_rn(t, s_all[q]);
    tol = kEps * sqrt(t);  // randomized.py:98, same summation order everywhere
  }

  int got = a.want;
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
  for (int j = 0; j < a.want; ++j) {
    const int par = j & 1;
    // ---- warp 0: winner (one key read) and the reflector (kernels.py:26-44)
    if (warp == 0) {
      const unsigned long long wk = slot_max(j % 3);
      const int owner = wk ? (int)omap[key_pos(wk, pb)] : -1;
      double xv[5];  // ell <= 160 (longer samples: the loop form below)
      double xnorm = -1.0;
      if (ell > 160) {
        // same arithmetic through shared memory: lane l sums rows l, l+32, ...
        // (ascending), then the warp tree -- the order of the register form
        const double* xc = nullptr;
        if (owner >= 0) {
          if constexpr (kCluster)
            xc = cg::this_cluster().map_shared_rank(ccol, owner) + par * cstride;
          else
            xc = a.gcol + ((size_t)par * P + owner) * cstride;
          for (int i = lane; i < ell; i += 32) vbuf[i] = kCluster ? xc[i] : __ldcg(xc + i);
          xnorm = kCluster ? xc[ell] : __ldcg(xc + ell);
        }
        __syncwarp();
        const bool halt = owner < 0 || !(xnorm > tol);  // qrcp.py:69-71
        if (!halt) {
          double sq = 0.0;
          for (int i = lane; i < ell; i += 32)
            if (i >= j) sq = __fma_rn(vbuf[i], vbuf[i], sq);
          sq = warp_sum(sq);
          const double alpha = vbuf[j];
          __syncwarp();
          const double norm = sqrt(sq);
          double beta = 0.0, tau = 0.0, den = 1.0;
          const bool zero = norm == 0.0;
          if (!zero) {
            beta = alpha >= 0.0 ? -norm : norm;
            den = __dsub_rn(alpha, beta);
            tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
          }
          const double rinv = zero ? 1.0 : __drcp_rn(den);
          for (int i = lane; i < ell; i += 32)
            if (i >= j) {
              const double v = (i == j) ? 1.0 : (zero ? vbuf[i] : __dmul_rn(vbuf[i], rinv));
              vbuf[i] = v;
              tvbuf[i] = __dmul_rn(tau, v);
            }
          if (lane == 0) {
            s_step[0] = beta;
            s_step[1] = tau;
          }
        }
        if (lane == 0) {
          s_stepi[0] = halt ? -1 : owner;
          s_stepi[1] = key_pos(wk, pb);
          if (!halt) {
            const int pp = key_pos(wk, pb);
            const unsigned char oj = omap[j];
            omap[j] = omap[pp];
            omap[pp] = oj;
          }
          s_bkey = 0ull;
          if constexpr (kCluster) {
            for (int q = 0; q < P; ++q) s_key[(j + 2) % 3][q] = 0ull;
          } else if (me == 0) {
            a.gkey[(j + 2) % 3] = 0ull;
          }
        }
      } else {   // ell <= 160: the column in registers
      if (owner >= 0) {
        const double* xc;
        if constexpr (kCluster) {
          xc = cg::this_cluster().map_shared_rank(ccol, owner) + par * cstride;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int i = lane + 32 * k;
            xv[k] = i < ell ? xc[i] : 0.0;
          }
          xnorm = xc[ell];
        } else {
          xc = a.gcol + ((size_t)par * P + owner) * cstride;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int i = lane + 32 * k;
            xv[k] = i < ell ? __ldcg(xc + i) : 0.0;
          }
          xnorm = __ldcg(xc + ell);
        }
      }
      const bool halt = owner < 0 || !(xnorm > tol);  // qrcp.py:69-71
      if (!halt) {
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int i = lane + 32 * k;
          if (i >= j && i < ell) sq = __fma_rn(xv[k], xv[k], sq);
        }
        sq = warp_sum(sq);
        double alpha = 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double t = __shfl_sync(0xffffffffu, xv[k], j & 31);
          if ((j >> 5) == k) alpha = t;
        }
        const double norm = sqrt(sq);
        double beta = 0.0, tau = 0.0, den = 1.0;
        const bool zero = norm == 0.0;
        if (!zero) {
          beta = alpha >= 0.0 ? -norm : norm;
          den = __dsub_rn(alpha, beta);
          tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
        }
        // v = x / (alpha - beta) (kernels.py:42) as x * (1/(alpha - beta)): one
        // division instead of one per row (<= 1 ulp from the reference's v)
        const double rinv = zero ? 1.0 : __drcp_rn(den);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int i = lane + 32 * k;
          if (i >= j && i < ell) {
            const double v = (i == j) ? 1.0 : (zero ? xv[k] : __dmul_rn(xv[k], rinv));
            vbuf[i] = v;
            tvbuf[i] = __dmul_rn(tau, v);
          }
        }
        if (lane == 0) {
          s_step[0] = beta;
          s_step[1] = tau;
        }
      }
      if (lane == 0) {
        s_stepi[0] = halt ? -1 : owner;
        s_stepi[1] = key_pos(wk, pb);
        if (!halt) {  // the swap j <-> p moves the owners too
          const int pp = key_pos(wk, pb);
          const unsigned char oj = omap[j];
          omap[j] = omap[pp];
          omap[pp] = oj;
        }
        s_bkey = 0ull;
        // recycle the slot read two steps ago (every CTA passed a sync since)
        if constexpr (kCluster) {
          for (int q = 0; q < P; ++q) s_key[(j + 2) % 3][q] = 0ull;
        } else if (me == 0) {
          a.gkey[(j + 2) % 3] = 0ull;
        }
      }
      }   // ell <= 160
    }
    __syncthreads();
    mark(0);
    const int owner = s_stepi[0], p = s_stepi[1];
    if (owner < 0) {
      got = j;
      break;
    }
    const double beta = s_step[0], tau = s_step[1];
    if (me == 0 && tid == 0) {
      a.piv[j] = p;
      if (a.taus) a.taus[j] = tau;
      const int64_t cols = (int64_t)a.nt - j - 1;
      if (tau != 0.0 && cols > 0) {
        l2 += 4LL * (ell - j) * cols;
        l2b += 16LL * (ell - j) * cols;
      }
    }
    if (me == 0 && a.Ys && warp == 0)
      for (int i = lane; i < ell; i += 32) a.Ys[(size_t)j * a.ldys + i] = i < j ? 0.0 : vbuf[i];
    mark(1);
    // ---- my columns, one 8-lane group per column: relabel (swap j <-> p),
    //      pivot column, apply H_j, downdate, next-step candidate key
    // each group keeps its best key of the step in a register; one shared
    // atomic per warp after the loop (a shared atomicMax per column made the
    // 64 groups of a CTA serialise on one address every step)
    unsigned long long gbest = 0ull;
    // this lane's rows j + gl + 8k of v, loaded once per step for all of its
    // columns (register form below); tau v is re-formed per use with the
    // same rounding as tvbuf
    double vk[20];
    if (ell <= 160) {
#pragma unroll
      for (int k = 0; k < 20; ++k) {
        const int r = j + gl + 8 * k;
        vk[k] = r < ell ? vbuf[r] : 0.0;
      }
    }
    for (int c = grp; c < ncol; c += NG) {
      double* col = colp(c);
      // read the column state before any lane of the group writes it
      int pc = pos[c];
      const double nv = nrm[c], og = orig[c];
      __syncwarp(gmask);
      if (pc == p) {
        // pivot column: rows < j keep R, row j = beta, below = 0 (qrcp.py:80-81)
        for (int i = j + gl; i < ell; i += 8) col[i] = (i == j) ? beta : 0.0;
        if (gl == 0) pos[c] = j;
        continue;
      }
      if (pc == j && p != j) {
        pc = p;
        if (gl == 0) pos[c] = p;
      }
      if (pc <= j) continue;
      if (ell <= 160) {
        // Register form: every row j + gl + 8k of the column is loaded before
        // any is used, so a column costs one memory round trip (the spilled
        // columns of wide samples live in L2/HBM: the loop form below waited
        // for one pair of loads per FMA step, ~37 us per pivot step on
        // cfg5's 136 x 32768 sample).  Arithmetic and order are the loop
        // form's: d0 takes rows j+gl+16q, d1 rows j+gl+8+16q, a lone tail
        // row goes to d0.
        double xr[20];
#pragma unroll
        for (int k = 0; k < 20; ++k) {
          const int r = j + gl + 8 * k;
          xr[k] = r < ell ? col[r] : 0.0;
        }
        if (tau != 0.0) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int k = 0; k < 20; k += 2) {
            const int r0 = j + gl + 8 * k;
            if (r0 + 8 < ell) {
              d0 = __fma_rn(vk[k], xr[k], d0);
              d1 = __fma_rn(vk[k + 1], xr[k + 1], d1);
            } else if (r0 < ell) {
              d0 = __fma_rn(vk[k], xr[k], d0);
            }
          }
          double w = __dadd_rn(d0, d1);
#pragma unroll
          for (int off = 4; off; off >>= 1) w = __dadd_rn(w, __shfl_xor_sync(gmask, w, off, 8));
#pragma unroll
          for (int k = 0; k < 20; ++k) {
            const int r = j + gl + 8 * k;
            if (r < ell) {
              xr[k] = __dsub_rn(xr[k], __dmul_rn(__dmul_rn(tau, vk[k]), w));
              col[r] = xr[k];
            }
          }
        }
        if (j + 1 < a.nt) {
          // NormTracker.downdate with row j (lane 0 of the group holds it)
          const double row = __shfl_sync(gmask, xr[0], 0, 8);
          double nsq = __dsub_rn(__dmul_rn(nv, nv), __dmul_rn(row, row));
          nsq = nsq > 0.0 ? nsq : 0.0;
          double nn;
          if (!(nsq < __dmul_rn(kGuard, og))) {
            nn = sqrt(nsq);
            if (gl == 0) nrm[c] = nn;
          } else {
            __syncwarp(gmask);   // the group's stores are visible
            double s0 = 0.0;
            for (int r = j + 1 + gl; r < ell; r += 8) s0 = __fma_rn(col[r], col[r], s0);
#pragma unroll
            for (int off = 4; off; off >>= 1) s0 = __dadd_rn(s0, __shfl_xor_sync(gmask, s0, off, 8));
            nn = sqrt(s0);
            if (gl == 0) {
              nrm[c] = nn;
              orig[c] = __dmul_rn(nn, nn);
            }
          }
          gbest = max(gbest, make_key(nn, pc, pb));
        }
        continue;
      }
      if (tau != 0.0) {
        double d0 = 0.0, d1 = 0.0;
        int i = j + gl;
        for (; i + 8 < ell; i += 16) {
          d0 = __fma_rn(vbuf[i], col[i], d0);
          d1 = __fma_rn(vbuf[i + 8], col[i + 8], d1);
        }
        if (i < ell) d0 = __fma_rn(vbuf[i], col[i], d0);
        double w = __dadd_rn(d0, d1);
#pragma unroll
        for (int off = 4; off; off >>= 1) w = __dadd_rn(w, __shfl_xor_sync(gmask, w, off, 8));
#pragma unroll 2
        for (int r = j + gl; r < ell; r += 8) col[r] = __dsub_rn(col[r], __dmul_rn(tvbuf[r], w));
      }
      double nn = nv;
      if (j + 1 < a.nt) {
        // NormTracker.downdate with row j of the updated sample (kernels.py:222-233)
        __syncwarp(gmask);
        const double row = col[j];
        double nsq = __dsub_rn(__dmul_rn(nv, nv), __dmul_rn(row, row));
        nsq = nsq > 0.0 ? nsq : 0.0;
        if (!(nsq < __dmul_rn(kGuard, og))) {
          nn = sqrt(nsq);
          if (gl == 0) nrm[c] = nn;
        } else {
          double s0 = 0.0;
          for (int r = j + 1 + gl; r < ell; r += 8) s0 = __fma_rn(col[r], col[r], s0);
#pragma unroll
          for (int off = 4; off; off >>= 1) s0 = __dadd_rn(s0, __shfl_xor_sync(gmask, s0, off, 8));
          nn = sqrt(s0);
          if (gl == 0) {
            nrm[c] = nn;
            orig[c] = __dmul_rn(nn, nn);
          }
        }
        gbest = max(gbest, make_key(nn, pc, pb));
      }
    }
    // warp max of the groups' keys (every lane of a group holds the same gbest)
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, gbest, off);
      gbest = o > gbest ? o : gbest;
    }
    if (lane == 0 && gbest != 0ull) atomicMax(&s_bkey, gbest);
    mark(2);
    publish((j + 1) % 3, par ^ 1);
    mark(3);
    xsync();
    mark(4);
  }
  if (timing) {
    for (int k = 0; k < 5; ++k) a.dbg[k] = tm[k];
    a.dbg[7] = a.want;
  }
  __syncthreads();
  // ---- write the transformed sample in pivoted order (group per column)
  for (int c = grp; c < ncol; c += NG) {
    const double* col = colp(c);
    double* dst = a.S + (size_t)pos[c] * a.lds;
    for (int i = gl; i < ell; i += 8) dst[i] = col[i];
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
  if constexpr (kCluster) cg::this_cluster().sync();  // peers may still read my smem
}

// v5: the same step with every column register-resident in its 8-lane group
// (lane gl holds rows gl, gl+8, ...; up to CPG columns per group) and the
// reflector formed redundantly by every warp (v, tau v in a per-warp shared
// slice), so a step has one block barrier plus the exchange and no shared
// memory round trips on the column path.  Same arithmetic rules as v4:
// reflector (kernels.py:26-44), H_j application, NormTracker downdate with
// the sqrt(eps) recompute guard (kernels.py:222-233), packed argmax key.
// v[idx] for a warp-uniform idx as a uniform branch (an unrolled compare-select
// chain is turned into a dynamically indexed local-memory array by the compiler)
template <int N>
RQ_DEV double pick_uniform(const double (&v)[N], int idx) {
  double out = v[0];
#define RQ_PICK(r) \
  case r:          \
    if constexpr (r < N) out = v[r]; \
    break;
  switch (idx) {
    RQ_PICK(1) RQ_PICK(2) RQ_PICK(3) RQ_PICK(4) RQ_PICK(5) RQ_PICK(6) RQ_PICK(7) RQ_PICK(8)
    RQ_PICK(9) RQ_PICK(10) RQ_PICK(11) RQ_PICK(12) RQ_PICK(13) RQ_PICK(14) RQ_PICK(15)
    RQ_PICK(16) RQ_PICK(17) RQ_PICK(18) RQ_PICK(19)
    default: break;
  }
#undef RQ_PICK
  return out;
}

template <bool kCluster, int RPL, int CPG>
__global__ void __launch_bounds__(kSelThreads, 1) select_reg_kernel(SelArgs a) {
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kSelThreads / 32;
  constexpr int NG = kSelThreads / 8;
  const int grp = tid >> 3, gl = tid & 7;
  const unsigned gmask = 0xffu << (lane & 24);  // my group's lanes
  int P, me;
  if constexpr (kCluster) {
    P = (int)cg::this_cluster().num_blocks();
    me = (int)cg::this_cluster().block_rank();
  } else {
    P = gridDim.x;
    me = blockIdx.x;
  }
  const int ell = a.ell, ldl = a.ldl;
  constexpr int pb = 16;   // register-resident samples are < 65536 columns wide (launch_select_reg)
  const int c0 = me * a.cpb;
  const int ncol = max(0, min(a.nt - c0, a.cpb));
  const int cstride = ell + 1;
  double* stage = sm;                                   // [cpb][ldl] initial load
  double* wv = stage + (size_t)a.cpb * ldl;             // [NW][ell] v
  double* wtv = wv + NW * ell;                          // [NW][ell] tau v
  double* ccol = wtv + NW * ell;                        // [2][ell+1] published candidate
  double* nrm0 = ccol + 2 * cstride;                    // [cpb] initial norms
  unsigned char* omap = (unsigned char*)(nrm0 + a.cpb); // [nt] position -> owner CTA
  __shared__ unsigned long long s_key[3][kMaxCluster];
  __shared__ unsigned long long s_wkey[2][NW];   // per-warp best keys, by step parity
  __shared__ double s_sq[kMaxCluster];
  __shared__ double s_all[160];
  __shared__ double s_step[2];
  __shared__ int s_stepi[2];
  unsigned int epoch = 0;
  auto xsync = [&]() {
    if constexpr (kCluster) cg::this_cluster().sync();
    else grid_barrier(a.bar, epoch);
  };
  __shared__ unsigned long long s_wk;
  const bool fused = !kCluster && a.pair != nullptr;
  // grid barrier whose arrival counter shares a 16-byte word with the step's
  // key slot: the acquire load that sees the last arrival has the final key
  // (every CTA's atomicMax precedes its fenced arrival; a .b128 load is one
  // scalar access in the PTX memory model, LDG.E.128.STRONG.GPU in SASS)
  auto fsync = [&](int slot) {
    __syncthreads();
    if (tid == 0) {
      ulonglong2* pr = a.pair + slot;
      __threadfence();
      atomicAdd((unsigned long long*)&pr->x, 1ull);
      unsigned long long c, k;
      do {
        asm volatile("{ .reg .b128 q; ld.acquire.gpu.global.b128 q, [%2]; mov.b128 {%0, %1}, q; }"
                     : "=l"(c), "=l"(k) : "l"(pr) : "memory");
      } while (c < (unsigned long long)P);
      s_wk = k;
    }
    __syncthreads();
  };
  auto slot_max = [&](int slot) -> unsigned long long {
    unsigned long long k = 0ull;
    if constexpr (kCluster) {
      if (lane < P) k = s_key[slot][lane];
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
        k = o > k ? o : k;
      }
    } else {
      k = fused ? s_wk : __ldcg(a.gkey + slot);
    }
    return k;
  };

  // ---- load, initial norms (pairwise, bit-identical to numpy), registers
  {
    const int total = ncol * ell;
#pragma unroll 4
    for (int e = tid; e < total; e += kSelThreads) {
      const int c = e / ell, i = e - c * ell;
      stage[(size_t)c * ldl + i] = a.B[(size_t)(c0 + c) * a.ldb + i];
    }
  }
  for (int e = tid; e < 3 * kMaxCluster; e += kSelThreads) (&s_key[0][0])[e] = 0ull;
  for (int q = tid; q < a.nt; q += kSelThreads) omap[q] = (unsigned char)(q / a.cpb);
  if (!kCluster && me == 0 && tid < 3) a.gkey[tid] = 0ull;
  __syncthreads();
  double mysq = 0.0;
  for (int c = tid; c < ncol; c += kSelThreads) {
    const double sq = pairwise_sumsq_256(stage + (size_t)c * ldl, ell, 1);   // ell <= 160 here
    nrm0[c] = sqrt(sq);
    mysq = __dadd_rn(mysq, sq);
  }
  {
    const double v = warp_sum(mysq);
    if (lane == 0) s_all[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t = __dadd_rn(t, s_all[w]);
      if constexpr (kCluster) {
        for (int q = 0; q < P; ++q) cg::this_cluster().map_shared_rank(s_sq, q)[me] = t;
      } else {
        a.gsq[me] = t;
      }
    }
  }
  double x[CPG][RPL];
  double nv[CPG], og[CPG];
  int pc[CPG];   // logical position of my column t (-1: none)
#pragma unroll
  for (int t = 0; t < CPG; ++t) {
    const int c = grp + NG * t;
    const bool valid = c < ncol;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = gl + 8 * r;
      x[t][r] = (valid && i < ell) ? stage[(size_t)c * ldl + i] : 0.0;
    }
    nv[t] = valid ? nrm0[c] : 0.0;
    og[t] = __dmul_rn(nv[t], nv[t]);
    pc[t] = valid ? c0 + c : -1;
  }
  if (!fused) xsync();  // key slots are zero everywhere before anyone publishes (fused: host memset)

  // publish the block's best candidate for step jn (key slot jn % 3, column
  // parity jn & 1); the caller has passed a block barrier since the keys
  auto publish = [&](int jn, unsigned long long bk) {
    if (bk == 0ull) return;
    if constexpr (kCluster) {
      if (tid < P) cg::this_cluster().map_shared_rank(&s_key[jn % 3][0], tid)[me] = bk;
    } else {
      if (tid == 0) atomicMax(fused ? (unsigned long long*)&a.pair[jn % 3].y : a.gkey + (jn % 3), bk);
    }
    const int bpos = key_pos(bk, pb);
#pragma unroll
    for (int t = 0; t < CPG; ++t) {
      if (pc[t] != bpos) continue;
      double* dst = kCluster ? ccol + (jn & 1) * cstride
                             : a.gcol + ((size_t)(jn & 1) * P + me) * cstride;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = gl + 8 * r;
        if (i < ell) dst[i] = x[t][r];
      }
      if (gl == 0) dst[ell] = nv[t];
    }
  };
  auto block_key = [&](int b) {   // max of the per-warp keys (every warp, after a barrier)
    unsigned long long k = lane < NW ? s_wkey[b][lane] : 0ull;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
      k = o > k ? o : k;
    }
    return k;
  };
  auto group_key = [&](unsigned long long k) {   // warp max of the groups' keys
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
      k = o > k ? o : k;
    }
    return k;
  };

  // step-0 candidates
  {
    unsigned long long k = 0ull;
#pragma unroll
    for (int t = 0; t < CPG; ++t) {
      if (pc[t] < 0) continue;
      const unsigned long long kt = make_key(nv[t], pc[t], pb);
      k = kt > k ? kt : k;
    }
    k = group_key(k);
    if (lane == 0) s_wkey[0][warp] = k;
    __syncthreads();
    publish(0, block_key(0));
  }
  if (fused) fsync(0);
  else xsync();
  double tol;
  {
    for (int q = tid; q < P; q += kSelThreads) {
      if constexpr (kCluster) s_all[q] = s_sq[q];
      else s_all[q] = a.gsq[q];
    }
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < P; ++q) t = __dadd_rn(t, s_all[q]);
    tol = kEps * sqrt(t);  // randomized.py:98, same summation order everywhere
  }

  int got = a.want;
  int64_t l2 = 0, l2b = 0;
  __shared__ long long tm[5];   // phase timers (thread 0 of CTA 0), off the register budget
  const bool timing = a.dbg != nullptr && me == 0 && tid == 0;
  if (timing) {
    for (int k = 0; k < 4; ++k) tm[k] = 0;
    tm[4] = clock64();
  }
  auto mark = [&](int k) {
    if (timing) {
      const long long t = clock64();
      tm[k] += t - tm[4];
      tm[4] = t;
    }
  };
  for (int j = 0; j < a.want; ++j) {
    const int par = j & 1;
    // ---- warp 0: winner and reflector into the shared v / tau v
    if (warp == 0) {
      const unsigned long long wk = slot_max(j % 3);
      const int pw = key_pos(wk, pb);
      const int owner = wk ? (int)omap[pw] : -1;
      double xv[5];  // ell <= 160
      double xnorm = -1.0;
      if (owner >= 0) {
        const double* xc;
        if constexpr (kCluster) {
          xc = cg::this_cluster().map_shared_rank(ccol, owner) + par * cstride;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int i = lane + 32 * k;
            xv[k] = i < ell ? xc[i] : 0.0;
          }
          xnorm = xc[ell];
        } else {
          xc = a.gcol + ((size_t)par * P + owner) * cstride;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const int i = lane + 32 * k;
            xv[k] = i < ell ? __ldcg(xc + i) : 0.0;
          }
          xnorm = __ldcg(xc + ell);
        }
      }
      const bool halt = owner < 0 || !(xnorm > tol);  // qrcp.py:69-71
      double beta = 0.0, tau = 0.0;
      if (!halt) {
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int i = lane + 32 * k;
          if (i >= j && i < ell) sq = __fma_rn(xv[k], xv[k], sq);
        }
        sq = warp_sum(sq);
        double alpha = 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double t = __shfl_sync(0xffffffffu, xv[k], j & 31);
          if ((j >> 5) == k) alpha = t;
        }
        const double norm = sqrt(sq);
        double den = 1.0;
        const bool zero = norm == 0.0;
        if (!zero) {
          beta = alpha >= 0.0 ? -norm : norm;
          den = __dsub_rn(alpha, beta);
          tau = __ddiv_rn(__dsub_rn(beta, alpha), beta);
        }
        const double rinv = zero ? 1.0 : __drcp_rn(den);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int i = lane + 32 * k;
          if (i >= j && i < ell) {
            wv[i] = (i == j) ? 1.0 : (zero ? xv[k] : __dmul_rn(xv[k], rinv));
          }
        }
      }
      if (lane == 0) {
        s_step[0] = beta;
        s_step[1] = tau;
        s_stepi[0] = halt ? -1 : owner;
        s_stepi[1] = pw;
      }
    }
    __syncthreads();
    if (s_stepi[0] < 0) {
      got = j;
      break;
    }
    const int p = s_stepi[1];
    const double beta = s_step[0], tau = s_step[1];
    if (me == 0 && warp == 0) {
      if (lane == 0) {
        a.piv[j] = p;
        if (a.taus) a.taus[j] = tau;
        const int64_t cols = (int64_t)a.nt - j - 1;
        if (tau != 0.0 && cols > 0) {
          l2 += 4LL * (ell - j) * cols;
          l2b += 16LL * (ell - j) * cols;
        }
      }
      if (a.Ys)
        for (int i = lane; i < ell; i += 32) a.Ys[(size_t)j * a.ldys + i] = i < j ? 0.0 : wv[i];
    }
    mark(0);
    // ---- my columns: relabel (swap j <-> p), pivot column, H_j, downdate, key
    double vr[RPL];   // tau v is formed per use (same rounding as wtv, fewer live registers)
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = gl + 8 * r;
      vr[r] = (i >= j && i < ell) ? wv[i] : 0.0;
    }
    unsigned long long key = 0ull;
    if constexpr (CPG > 1) {
      // Several columns per group: the same arithmetic per column as the
      // one-column form below, but phase by phase over the columns (dot
      // products, reductions, updates, norms), without per-column branches,
      // so the columns' dependent chains overlap.  Inactive columns (pivoted
      // ones, the pivot itself, empty slots) run the arithmetic too and
      // discard it.
      int qq[CPG];
      bool act[CPG], isp[CPG];
#pragma unroll
      for (int t = 0; t < CPG; ++t) {
        int q = pc[t];
        isp[t] = q >= 0 && q == p;
        if (!isp[t] && q == j && p != j) {
          q = p;
          pc[t] = p;
        }
        act[t] = !isp[t] && q > j;
        qq[t] = q;
      }
      if (tau != 0.0) {
        double w[CPG];
#pragma unroll
        for (int t = 0; t < CPG; ++t) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int r = 0; r < RPL; r += 2) {
            d0 = __fma_rn(vr[r], x[t][r], d0);
            if (r + 1 < RPL) d1 = __fma_rn(vr[r + 1], x[t][r + 1], d1);
          }
          w[t] = __dadd_rn(d0, d1);
        }
#pragma unroll
        for (int off = 4; off; off >>= 1)
#pragma unroll
          for (int t = 0; t < CPG; ++t)
            w[t] = __dadd_rn(w[t], __shfl_xor_sync(0xffffffffu, w[t], off, 8));
#pragma unroll
        for (int t = 0; t < CPG; ++t)
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = gl + 8 * r;
            if (act[t] && i >= j) x[t][r] = __dsub_rn(x[t][r], __dmul_rn(__dmul_rn(tau, vr[r]), w[t]));
          }
      }
#pragma unroll
      for (int t = 0; t < CPG; ++t) {
        if (!isp[t]) continue;
        // pivot column: rows < j keep R, row j = beta, below = 0 (qrcp.py:80-81)
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = gl + 8 * r;
          if (i == j) x[t][r] = beta;
          else if (i > j) x[t][r] = 0.0;
        }
        pc[t] = j;
      }
      if (j + 1 < a.nt) {
        // NormTracker.downdate with row j of the updated sample (kernels.py:222-233)
        double nn[CPG];
        bool rec[CPG];
#pragma unroll
        for (int t = 0; t < CPG; ++t) {
          const double rsel = pick_uniform<RPL>(x[t], j >> 3);
          const double row = __shfl_sync(0xffffffffu, rsel, j & 7, 8);
          double nsq = __dsub_rn(__dmul_rn(nv[t], nv[t]), __dmul_rn(row, row));
          nsq = nsq > 0.0 ? nsq : 0.0;
          rec[t] = act[t] && nsq < __dmul_rn(kGuard, og[t]);
          nn[t] = sqrt(nsq);
        }
#pragma unroll
        for (int t = 0; t < CPG; ++t) {
          if (!rec[t]) continue;   // (uniform over the group: its lanes share the column)
          double s0 = 0.0;
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = gl + 8 * r;
            if (i > j && i < ell) s0 = __fma_rn(x[t][r], x[t][r], s0);
          }
#pragma unroll
          for (int off = 4; off; off >>= 1) s0 = __dadd_rn(s0, __shfl_xor_sync(gmask, s0, off, 8));
          nn[t] = sqrt(s0);
          og[t] = __dmul_rn(nn[t], nn[t]);
        }
#pragma unroll
        for (int t = 0; t < CPG; ++t) {
          if (!act[t]) continue;
          nv[t] = nn[t];
          const unsigned long long kt = make_key(nn[t], qq[t], pb);
          key = kt > key ? kt : key;
        }
      }
    } else {
#pragma unroll
    for (int t = 0; t < CPG; ++t) {
      int q = pc[t];
      if (q < 0) continue;
      if (q == p) {
        // pivot column: rows < j keep R, row j = beta, below = 0 (qrcp.py:80-81)
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = gl + 8 * r;
          if (i == j) x[t][r] = beta;
          else if (i > j) x[t][r] = 0.0;
        }
        pc[t] = j;
        continue;
      }
      if (q == j && p != j) {
        q = p;
        pc[t] = p;
      }
      if (q <= j) continue;
      if (tau != 0.0) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; r += 2) {
          d0 = __fma_rn(vr[r], x[t][r], d0);
          if (r + 1 < RPL) d1 = __fma_rn(vr[r + 1], x[t][r + 1], d1);
        }
        double w = __dadd_rn(d0, d1);
#pragma unroll
        for (int off = 4; off; off >>= 1) w = __dadd_rn(w, __shfl_xor_sync(gmask, w, off, 8));
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = gl + 8 * r;
          if (i >= j) x[t][r] = __dsub_rn(x[t][r], __dmul_rn(__dmul_rn(tau, vr[r]), w));
        }
      }
      if (j + 1 < a.nt) {
        // NormTracker.downdate with row j of the updated sample (kernels.py:222-233)
        const double rsel = pick_uniform<RPL>(x[t], j >> 3);
        const double row = __shfl_sync(gmask, rsel, j & 7, 8);
        double nsq = __dsub_rn(__dmul_rn(nv[t], nv[t]), __dmul_rn(row, row));
        nsq = nsq > 0.0 ? nsq : 0.0;
        double nn;
        if (!(nsq < __dmul_rn(kGuard, og[t]))) {
          nn = sqrt(nsq);
        } else {
          double s0 = 0.0;
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = gl + 8 * r;
            if (i > j && i < ell) s0 = __fma_rn(x[t][r], x[t][r], s0);
          }
#pragma unroll
          for (int off = 4; off; off >>= 1) s0 = __dadd_rn(s0, __shfl_xor_sync(gmask, s0, off, 8));
          nn = sqrt(s0);
          og[t] = __dmul_rn(nn, nn);
        }
        nv[t] = nn;
        const unsigned long long kt = make_key(nn, q, pb);
        key = kt > key ? kt : key;
      }
    }
    }   // CPG == 1
    key = group_key(key);
    if (lane == 0) s_wkey[par ^ 1][warp] = key;
    mark(1);
    __syncthreads();   // block keys complete; every warp is past its omap reads of step j
    const unsigned long long bk = block_key(par ^ 1);
    if (tid == 0) {
      // the swap j <-> p moves the owners too
      const unsigned char oj = omap[j];
      omap[j] = omap[p];
      omap[p] = oj;
      // recycle the key slot read at step j - 1 (every CTA passed an exchange since)
      if constexpr (kCluster) {
        for (int q = 0; q < P; ++q) s_key[(j + 2) % 3][q] = 0ull;
      } else if (me == 0) {
        if (fused) a.pair[(j + 2) % 3] = make_ulonglong2(0ull, 0ull);
        else a.gkey[(j + 2) % 3] = 0ull;
      }
    }
    publish(j + 1, bk);
    mark(2);
    if (fused) fsync((j + 1) % 3);
    else xsync();
    mark(3);
  }
  if (timing) {
    for (int k = 0; k < 4; ++k) a.dbg[k] = tm[k];
    a.dbg[7] = a.want;
  }
  // ---- transformed sample in pivoted order
#pragma unroll
  for (int t = 0; t < CPG; ++t) {
    if (pc[t] < 0) continue;
    double* dst = a.S + (size_t)pc[t] * a.lds;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = gl + 8 * r;
      if (i < ell) dst[i] = x[t][r];
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
  if constexpr (kCluster) cg::this_cluster().sync();  // peers may still read my smem
}


template <bool kCluster, int RPL, int CPG>
void launch_reg(Handle& h, int P, size_t smem, SelArgs& a, cudaStream_t s) {
  auto kern = select_reg_kernel<kCluster, RPL, CPG>;
  if (kCluster) kernel_attr((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  kernel_attr((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)std::max<size_t>(smem, 48 * 1024));
  if constexpr (!kCluster) {
    void* args[] = {&a};
    RQ_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(P), dim3(kSelThreads), args, smem, s));
  } else {
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
    RQ_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  }
}

// v5 (register-resident columns) when the CTA's columns fit its 64 groups
// twice and the sample rows fit the per-lane register budget
bool launch_select_reg(Handle& h, bool grid, int P, int cpb, int64_t ell, int64_t nt,
                       int64_t want, const double* B, int64_t ldb, const SelectOut& out,
                       Status* st, bool abort_on_short, int64_t i0, cudaStream_t s) {
  constexpr int NG = kSelThreads / 8, NW = kSelThreads / 32;
  const int cpg = cpb <= NG ? 1 : (cpb <= 2 * NG ? 2 : (cpb <= 3 * NG ? 3 : 0));
  const int rpl = ell <= 40 ? 5 : (ell <= 72 ? 9 : (ell <= 136 ? 17 : (ell <= 160 ? 20 : 0)));
  if (cpg == 0 || rpl == 0 || (rpl > 9 && cpg > 1) || nt > 65535) return false;
  const int ldl = (int)(ell | 1);
  const size_t smem = ((size_t)cpb * ldl + 2 * (size_t)NW * ell + 2 * (ell + 1) + cpb) * 8 +
                      (size_t)nt + 64;
  if (smem > h.smem_optin) return false;
  SelArgs a{};
  a.ell = (int)ell; a.nt = (int)nt; a.want = (int)want;
  a.pbits = nt > 65535 ? 20 : 16;
  a.abort_on_short = abort_on_short ? 1 : 0;
  a.i0 = i0;
  a.B = B; a.ldb = ldb;
  a.S = out.S; a.lds = out.lds; a.piv = out.piv; a.Ys = out.Ys; a.ldys = out.ldys;
  a.taus = out.taus;
  a.st = st;
  a.cpb = cpb; a.ldl = ldl; a.ncs = cpb;
  a.dbg = h.dbg;
  ProfScope prof(h, kProfSelect, 4.0 * ell * nt * want, 16.0 * ell * nt, s);
  count_launch();
  if (grid) {
    a.bar = (unsigned int*)h.buf("sel_bar", 128, s);
    a.gkey = (unsigned long long*)h.buf("sel_gkey", 64, s);
    a.gcol = (double*)h.buf("sel_gcol", (size_t)2 * P * (ell + 1) * 8, s);
    a.gsq = (double*)h.buf("sel_gsq", (size_t)P * 8, s);
    a.pair = h.select_fused ? (ulonglong2*)((char*)a.bar + 64) : nullptr;
    RQ_CUDA(cudaMemsetAsync(a.bar, 0, 128, s));
  }
#define RQ_SEL_REG(R, C)                                                   \
  if (rpl == R && cpg == C) {                                             \
    if (grid) launch_reg<false, R, C>(h, P, smem, a, s);                  \
    else launch_reg<true, R, C>(h, P, smem, a, s);                        \
    return true;                                                          \
  }
  RQ_SEL_REG(5, 1) RQ_SEL_REG(5, 2) RQ_SEL_REG(5, 3) RQ_SEL_REG(9, 1) RQ_SEL_REG(9, 2)
  RQ_SEL_REG(9, 3) RQ_SEL_REG(17, 1)
  RQ_SEL_REG(20, 1)
#undef RQ_SEL_REG
  return false;
}

}  // namespace

void select_pivots(Handle& h, int64_t ell, int64_t nt, int64_t want, const double* B,
                   int64_t ldb, const SelectOut& out, Status* st, bool abort_on_short,
                   int64_t i0, cudaStream_t s, int max_ctas) {
  if (want < 1 || want > std::min(ell, nt))
    throw InvalidArg("cannot select " + std::to_string(want) + " pivots from a " +
                     std::to_string(ell) + " x " + std::to_string(nt) + " sample");
  if (ell > 4096) throw InvalidArg("sample rows > 4096 not supported by the pivot kernel");
  if (nt >= (1 << 20)) throw InvalidArg("sample wider than 2^20 - 1 columns");
  const bool grid = h.force_select == 1 ||
                    (h.force_select == 0 && nt > h.select_cluster_max_cols);
  int P;
  if (grid) {
    int cap = h.select_max_ctas > 0 ? std::min(h.select_max_ctas, h.num_sms) : h.num_sms;
    if (max_ctas > 0) cap = std::min(cap, max_ctas);
    P = (int)std::min<int64_t>(std::min(cap, 160), (nt + 31) / 32);  // owner ids fit a byte
    P = std::max(P, 1);
    const int cpb = (int)((nt + P - 1) / P);
    P = (int)((nt + cpb - 1) / cpb);
  } else {
    P = 1;
    while (P < kMaxCluster && (int64_t)P * 64 < nt) P <<= 1;
  }
  const int cpb = (int)((nt + P - 1) / P);
  if (cpb > 8192) throw InvalidArg("sample too wide for the pivot kernel");
  if (h.select_reg && launch_select_reg(h, grid, P, cpb, ell, nt, want, B, ldb, out, st,
                                        abort_on_short, i0, s))
    return;
  const int ldl = (int)(ell | 1);
  const size_t meta = ((size_t)2 * ell + 2 * (ell + 1) + 2 * (size_t)cpb + 16) * 8 +
                      (size_t)cpb * 4 + (size_t)nt + 256;
  const size_t colbytes = (size_t)ldl * 8;
  const int ncs = (int)std::min<size_t>(cpb, (h.smem_optin - 4096 - meta) / colbytes);
  const size_t smem = (size_t)ncs * colbytes + meta;
  SelArgs a{};
  a.ell = (int)ell; a.nt = (int)nt; a.want = (int)want;
  a.pbits = nt > 65535 ? 20 : 16;
  a.abort_on_short = abort_on_short ? 1 : 0;
  a.i0 = i0;
  a.B = B; a.ldb = ldb;
  a.S = out.S; a.lds = out.lds; a.piv = out.piv; a.Ys = out.Ys; a.ldys = out.ldys;
  a.taus = out.taus;
  a.st = st;
  a.gstore = ncs < cpb ? (double*)h.buf("sel_gstore", (size_t)P * (cpb - ncs) * colbytes, s)
                       : nullptr;
  a.cpb = cpb; a.ldl = ldl; a.ncs = ncs;
  a.dbg = h.dbg;
  ProfScope prof(h, kProfSelect, 4.0 * ell * nt * want, 16.0 * ell * nt, s);
  count_launch();
  if (grid) {
    a.bar = (unsigned int*)h.buf("sel_bar", 128, s);
    a.gkey = (unsigned long long*)h.buf("sel_gkey", 64, s);
    a.gcol = (double*)h.buf("sel_gcol", (size_t)2 * P * (ell + 1) * 8, s);
    a.gsq = (double*)h.buf("sel_gsq", (size_t)P * 8, s);
    RQ_CUDA(cudaMemsetAsync(a.bar, 0, 64, s));
    kernel_attr((const void*)select_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)std::max<size_t>(smem, 48 * 1024));
    void* args[] = {&a};
    RQ_CUDA(cudaLaunchCooperativeKernel((void*)select_kernel<false>, dim3(P), dim3(kSelThreads),
                                        args, smem, s));
    return;
  }
  kernel_attr((const void*)select_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  kernel_attr((const void*)select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
              (int)std::max<size_t>(smem, 48 * 1024));
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
  RQ_CUDA(cudaLaunchKernelEx(&cfg, select_kernel<true>, a));
}

}  // namespace rq
