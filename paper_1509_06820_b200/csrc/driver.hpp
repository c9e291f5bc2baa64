// Native drivers for the randomized QRCP family (driver.cu).
#pragma once

#include "runtime.hpp"

namespace rq {

// host Omega source: fill host_dst (rows x cols, column-major) with the next
// rows*cols draws of the caller's RngState stream (rng.py:36-41).
typedef int (*OmegaFn)(void* user, int64_t rows, int64_t cols, double* host_dst);

struct Counters {
  int64_t gemm_flops = 0, level2_flops = 0, bytes_touched = 0, resamples = 0;
};

struct FactorParams {
  int64_t m = 0, n = 0, k = 0;   // k validated, 1 <= k <= min(m, n)
  int64_t block = 32;            // pivot block width (ssrqrcp: k)
  int64_t ell = 40;              // sample rows (ssrqrcp: k + padding)
  int resketch_each_block = 0;   // rsrqrcp
  int update_trailing = 1;       // 0: ssrqrcp (R rows only)
  int truncated = 0;             // 1: TRQRCP (no trailing update, W panel)
  double* work = nullptr; int64_t ldw = 0;   // in: copy of A; out (RQRCP): R rows + trailing
  double* Y = nullptr; int64_t ldy = 0;      // m x k, out
  double* tau = nullptr;                     // k, out
  double* W = nullptr; int64_t ldW = 0;      // TRQRCP: n x k inner-product panel, out
  double* R = nullptr; int64_t ldR = 0;      // TRQRCP: k x n, out
  int64_t* perm = nullptr;                   // n, out (forward map)
  int64_t* swaps = nullptr; int64_t swap_cap = 0;  // 2*swap_cap int64, out
  const double* omega0 = nullptr;            // optional explicit first Omega (device, ell x m)
  OmegaFn omega_fn = nullptr;
  void* omega_user = nullptr;
  int speculate = 1;                         // 0: synchronise every block (debug)
  cudaStream_t stream = nullptr;
  double* host_Y = nullptr; int64_t ldhY = 0;   // optional pinned outputs streamed as blocks commit
  double* host_R = nullptr; int64_t ldhR = 0;
  bool omega_native = false;                  // draw with rq_omega_fill (key, raw) instead of omega_fn
  int omega_threads = 1;
  uint64_t omega_k0 = 0, omega_k1 = 0, omega_raw = 0;
};

struct FactorResult {
  int64_t rank = 0, nswaps = 0;
  Counters c;
  double frob = 0.0;
};

FactorResult run_factor(Handle& h, const FactorParams& p);

// unpivoted blocked QR in place (qrcp.py:222-252): Y (m x k), tau, R = work[:k,:]
void qr_blocked(Handle& h, int64_t m, int64_t n, int64_t k, int64_t b, double* work,
                int64_t ldw, double* Y, int64_t ldy, double* tau, Counters* c, cudaStream_t s);
// leading `cols` columns of I - Y T Y^T (qrcp.py:53-60), blocked backward
// accumulation with block width b
void q_columns(Handle& h, int64_t m, int64_t nref, int64_t cols, const double* Y, int64_t ldy,
               const double* tau, int64_t b, double* Q, int64_t ldq, cudaStream_t s);

}  // namespace rq

namespace rq {

struct TuxvParams {
  FactorParams f;               // truncated = 1; f.work is a scratch copy of A
  const double* A = nullptr; int64_t lda = 0;   // original A (device, not modified)
  int64_t j_max = 1;
  double* U = nullptr; int64_t ldu = 0;         // m x k
  double* V = nullptr; int64_t ldv = 0;         // n x k
  double* X = nullptr; int64_t ldx = 0;         // k x k
};
struct TuxvResult {
  FactorResult f;
  int64_t rank = 0;
  int x_lower = 0;   // 1 when the last half-iteration was an LQ (X lower triangular)
};
// truncated.py:208-252 (without svd_of_x, which the host applies on the k x k core)
TuxvResult run_tuxv(Handle& h, const TuxvParams& p);

}  // namespace rq
