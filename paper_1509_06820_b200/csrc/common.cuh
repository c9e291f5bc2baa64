// Shared device helpers for the sm_100a RQRCP kernels.
//
// Layout conventions: every matrix is FP64,
// column-major with an explicit leading dimension; permutations and swap logs
// are int64.  Kernels on the speculative block path take `abort`, a device
// word that, once non-zero, turns every later kernel of the queue into a
// no-op (see driver.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define RQ_DEV __device__ __forceinline__

namespace rq {

constexpr double kEps = 2.220446049250313e-16;         // np.finfo(float64).eps
constexpr double kGuard = 1.4901161193847656e-08;      // sqrt(eps), kernels.py:205
constexpr double kEps34 = 1.8189894035458565e-12;      // eps**0.75 = 2^-39, randomized.py:117

// abort codes written by the speculative-path kernels (driver.cu)
enum AbortCode : int {
  kAbortNone = 0,
  kAbortShortSample = 1,  // select: got < want   (randomized.py:217)
  kAbortPanelRank = 2,    // panel: usable < got  (randomized.py:229)
  kAbortDegenerate = 3,   // sample update: |R11_jj| < eps^3/4 ||A|| (randomized.py:117)
  kAbortPanelFast = 4,    // fast panel declined: redo this block's panel column by column
};

// Device-side run status shared by the kernels of one driver call.
struct Status {
  int abort;        // AbortCode of the first failing stage (0 = none)
  int pad0;
  int64_t abort_i0; // block start of the failing stage
  int64_t got;      // last select_pivots result
  int64_t usable;   // last panel rank
  int64_t level2;   // level-2 flop counter (OpCounters.level2_flops)
  int64_t l2bytes;  // bytes_touched contribution of the level-2 calls
  int64_t nswaps;   // length of the global swap log
  int64_t degenerate;  // last sample-update verdict (1 = degenerate)
};

RQ_DEV int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
RQ_DEV int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

RQ_DEV bool aborted(const Status* st) {
  return st != nullptr && *((volatile const int*)&st->abort) != 0;
}

// Software grid barrier for cooperative launches (all CTAs co-resident).
// `counter` must be zero at launch; `epoch` is a per-CTA register.
RQ_DEV void grid_barrier(unsigned int* counter, unsigned int& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += 1;
    const unsigned int target = epoch * gridDim.x;
    __threadfence();
    atomicAdd(counter, 1u);
    unsigned int seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
    } while (seen < target);
  }
  __syncthreads();
}

// Same barrier for waits that can be long (the other CTAs idle while one CTA
// runs a serial section): after a few fast polls the waiting thread backs off
// with __nanosleep, so ~150 pollers do not saturate the L2 slice that holds
// the counter (and with it the working CTA's own global traffic).
RQ_DEV void grid_barrier_patient(unsigned int* counter, unsigned int& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += 1;
    const unsigned int target = epoch * gridDim.x;
    __threadfence();
    atomicAdd(counter, 1u);
    unsigned int seen, ns = 32;
    int polls = 0;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
      if (seen >= target) break;
      if (++polls > 16) {
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;
      }
    }
  }
  __syncthreads();
}

// The patient barrier in two halves: a CTA that has published what the others
// wait for arrives, keeps working on results nobody reads inside the kernel,
// and waits afterwards.
RQ_DEV void grid_barrier_arrive(unsigned int* counter, unsigned int& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += 1;
    __threadfence();
    atomicAdd(counter, 1u);
  }
}
RQ_DEV void grid_barrier_wait(unsigned int* counter, const unsigned int& epoch) {
  if (threadIdx.x == 0) {
    const unsigned int target = epoch * gridDim.x;
    unsigned int seen, ns = 32;
    int polls = 0;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
      if (seen >= target) break;
      if (++polls > 16) {
        __nanosleep(ns);
        ns = ns < 512 ? 2 * ns : 512;
      }
    }
  }
  __syncthreads();
}

// numpy's pairwise summation (pairwise_sum_DOUBLE: 8 accumulators for
// n <= 128, recursive halving on multiples of 8 above) of x[i]*x[i] over a
// strided vector; bit-identical to np.linalg.norm(B, axis=0)**2 on an
// F-ordered sample (kernels.py:184-186, 207-209).
RQ_DEV double pairwise_block_sumsq(const double* x, int n, int stride) {
  double res;
  if (n < 8) {
    res = 0.0;
    for (int i = 0; i < n; ++i) {
      const double v = x[i * stride];
      res = __dadd_rn(res, __dmul_rn(v, v));
    }
    return res;
  }
  double r[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const double v = x[t * stride];
    r[t] = __dmul_rn(v, v);
  }
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double v = x[(i + t) * stride];
      r[t] = __dadd_rn(r[t], __dmul_rn(v, v));
    }
  }
  res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                  __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) {
    const double v = x[i * stride];
    res = __dadd_rn(res, __dmul_rn(v, v));
  }
  return res;
}

// n <= 256: one split at most (the register-resident pivot kernel's samples)
__device__ inline double pairwise_sumsq_256(const double* x, int n, int stride) {
  if (n <= 128) return pairwise_block_sumsq(x, n, stride);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_block_sumsq(x, n2, stride),
                   pairwise_block_sumsq(x + (size_t)n2 * stride, n - n2, stride));
}

// numpy's recursion (left half n2 = n/2 rounded down to a multiple of 8, then
// the rest) as an explicit post-order walk: device recursion would need a
// call stack the launch cannot size (samples taller than 1024 rows overflowed
// the default one)
__device__ inline double pairwise_sumsq(const double* x, int n, int stride) {
  if (n <= 128) return pairwise_block_sumsq(x, n, stride);
  constexpr int kDepth = 24;   // n halves per level down to <= 128: 2^31 needs 24
  int off[kDepth], len[kDepth], stage[kDepth];
  double left[kDepth];
  int sp = 0;
  off[0] = 0; len[0] = n; stage[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    if (stage[sp] == 0) {
      if (len[sp] <= 128) {
        ret = pairwise_block_sumsq(x + (size_t)off[sp] * stride, len[sp], stride);
        --sp;
      } else {
        int n2 = len[sp] / 2;
        n2 -= n2 % 8;
        stage[sp] = 1;
        off[sp + 1] = off[sp]; len[sp + 1] = n2; stage[sp + 1] = 0;
        ++sp;
      }
    } else if (stage[sp] == 1) {
      left[sp] = ret;
      int n2 = len[sp] / 2;
      n2 -= n2 % 8;
      stage[sp] = 2;
      off[sp + 1] = off[sp] + n2; len[sp + 1] = len[sp] - n2; stage[sp + 1] = 0;
      ++sp;
    } else {
      ret = __dadd_rn(left[sp], ret);
      --sp;
    }
  }
  return ret;
}

}  // namespace rq
