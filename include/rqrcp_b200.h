/* C-ABI of the B200-native randomized QRCP library (librqrcp_b200.so).
 *
 * The reference (arxiv 1509.06820, package `rqrcp` 0.1.0) has no FFI: its
 * operator API is the Python signatures of pkg/src/rqrcp/{randomized,
 * truncated,qrcp,kernels}.py.  Each entry point below replaces the named
 * reference function for device-resident FP64 data; the Python host layer
 * (paper_1509_06820_b200/) binds them with ctypes and keeps the reference
 * signatures.  INTEGRATION.md shows the binding.
 *
 * Conventions: all matrices are FP64, column-major, with explicit leading
 * dimensions; every pointer argument named A/B/C/Y/... is a DEVICE pointer
 * unless documented as host; `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Functions return 0 on success, RQ_ERR_INVALID for
 * argument errors (the reference's ValueError), RQ_ERR_CUDA for CUDA
 * failures and RQ_ERR_INTERNAL otherwise; rq_last_error() describes the last
 * failure of the calling thread.  A handle is bound to one device and is not
 * thread-safe; calls on one handle are stream-ordered.
 */
#ifndef RQRCP_B200_H
#define RQRCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RQ_OK 0
#define RQ_ERR_INVALID -1
#define RQ_ERR_INTERNAL -2
#define RQ_ERR_CUDA -3

typedef struct rq_handle_s* rq_handle_t;

/* library version (major*10000 + minor*100 + patch) */
int rq_version(void);
/* message of the last failing call on this thread ("" if none) */
const char* rq_last_error(void);

int rq_create(int device, rq_handle_t* out);
int rq_destroy(rq_handle_t h);

/* Host Omega source: write rows*cols i.i.d. N(0,1) draws, column-major, into
 * host_dst (the next draws of the caller's RngState stream, rng.py:16-41).
 * Return 0 on success. */
typedef int (*rq_omega_fn)(void* user, int64_t rows, int64_t cols, double* host_dst);

/* ---------------------------------------------------------------- drivers */

enum rq_variant {
  RQ_RQRCP = 0,   /* rqrcp    randomized.py:269-281 */
  RQ_RSRQRCP = 1, /* rsrqrcp  randomized.py:284-296 */
  RQ_SSRQRCP = 2, /* ssrqrcp  randomized.py:299-313 */
  RQ_TRQRCP = 3   /* trqrcp   truncated.py:70-174  */
};

typedef struct {
  int64_t m, n;        /* A is m x n */
  int64_t k;           /* validated rank, 1 <= k <= min(m, n) */
  int64_t block;       /* pivot block width b (ssrqrcp: k) */
  int64_t ell;         /* sample rows b + p (ssrqrcp: k + p) */
  int32_t variant;     /* enum rq_variant */
  int32_t speculate;   /* 1: no host sync between blocks (default); 0: debug */
  double* work;        /* in: copy of A (m x n, ldw); out: R rows (+ trailing) */
  int64_t ldw;
  double* Y;           /* out: m x k unit-lower reflectors */
  int64_t ldy;
  double* tau;         /* out: k */
  double* W;           /* TRQRCP out: n x k inner-product panel (else NULL) */
  int64_t ldW;
  double* R;           /* TRQRCP out: k x n R rows (else NULL) */
  int64_t ldR;
  int64_t* perm;       /* out: n, Permutation.forward */
  int64_t* swaps;      /* out: 2 * swap_cap int64 (pairs), Permutation.swaps */
  int64_t swap_cap;
  const double* omega0;  /* optional explicit first Omega (device, ell x m, ld ell) */
  rq_omega_fn omega_fn;  /* host Omega stream for (re)samples */
  void* omega_user;
  void* stream;
  /* optional host (pinned) outputs, filled while the factorization runs: the
   * columns of Y (m x k) and of R (k x n; RQRCP: work rows 0..k-1) are
   * streamed out as their blocks commit (later blocks never touch them) */
  double* host_Y;
  int64_t ldhY;
  double* host_R;
  int64_t ldhR;
  /* optional native Omega stream: when omega_native = 1 the (re)sample draws
   * come from rq_omega_fill on the caller's Philox key (omega_k0, omega_k1)
   * from raw counter omega_raw, on omega_threads host threads, instead of
   * omega_fn -- no callback into the caller, so they can be drawn ahead on a
   * host thread while the factorization runs */
  int32_t omega_native;
  int32_t omega_threads;
  uint64_t omega_k0, omega_k1, omega_raw;
} rq_factor_args;

typedef struct {
  int64_t rank;
  int64_t nswaps;
  int64_t gemm_flops, level2_flops, bytes_touched, resamples; /* OpCounters */
  double frob;         /* ||A||_F as computed on the device */
} rq_factor_result;

/* rqrcp / rsrqrcp / ssrqrcp / trqrcp (randomized.py:183-266,
 * truncated.py:70-174).  Synchronous: returns after the factorization. */
int rq_factor(rq_handle_t h, const rq_factor_args* args, rq_factor_result* out);

typedef struct {
  rq_factor_args f;    /* variant must be RQ_TRQRCP; f.work = scratch copy of A */
  const double* A;     /* original A, m x n (not modified) */
  int64_t lda;
  int64_t j_max;
  double* U; int64_t ldu;  /* out: m x k */
  double* V; int64_t ldv;  /* out: n x k */
  double* X; int64_t ldx;  /* out: k x k */
} rq_tuxv_args;

typedef struct {
  rq_factor_result f;
  int64_t rank;
  int32_t x_lower;
  int32_t pad;
} rq_tuxv_result;

/* tuxv (truncated.py:208-252) without the optional svd_of_x rotation. */
int rq_tuxv(rq_handle_t h, const rq_tuxv_args* args, rq_tuxv_result* out);

/* ---------------------------------------------------------------- primitives */

/* C = alpha op(A) op(B) + beta C (FP64 DMMA); transa/transb: 0 = N, 1 = T */
int rq_gemm(rq_handle_t h, int transa, int transb, int64_t m, int64_t n, int64_t k,
            double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
            double beta, double* C, int64_t ldc, void* stream);

/* make_sample core: B (ell x n) = Omega (ell x m) A (m x n)  (randomized.py:69-82) */
int rq_sketch(rq_handle_t h, int64_t ell, int64_t m, int64_t n, const double* omega,
              int64_t ldo, const double* A, int64_t lda, double* B, int64_t ldb, void* stream);

/* select_pivots (randomized.py:85-104): `want` greedy pivoted Householder
 * steps on the ell x nt sample B (not modified).  Outputs: S = transformed
 * sample in pivoted order (ell x nt), piv[j] = local column swapped with j
 * at step j, optional sample reflectors Ys (ell x want) / taus (want).
 * Synchronous; *got and *level2 (host) receive the step count and the
 * level-2 flop count. */
int rq_select_pivots(rq_handle_t h, int64_t ell, int64_t nt, int64_t want, const double* B,
                     int64_t ldb, double* S, int64_t lds, int64_t* piv, double* Ys,
                     int64_t ldys, double* taus, int64_t* got, int64_t* level2,
                     void* stream);

/* panel_householder + _panel_rank + build_t_matrix (qrcp.py:206-219,
 * randomized.py:150-155, kernels.py:139-147): in-place Householder QR of the
 * mm x bw panel P (R in the upper triangle, zeros below), reflectors into
 * Y (mm x bw), tau, and T (bw x bw, may be NULL).  tol < 0 disables the rank
 * test.  Synchronous; *usable and *level2 are host outputs. */
int rq_panel_qr(rq_handle_t h, int64_t mm, int64_t bw, double* P, int64_t ldp, double* Y,
                int64_t ldy, double* tau, double* T, int64_t ldt, double tol, int64_t* usable,
                int64_t* level2, void* stream);

/* build_t_matrix (kernels.py:139-147) for Y (mm x nb) */
int rq_t_factor(rq_handle_t h, const double* Y, int64_t ldy, int64_t mm, int64_t nb,
                const double* tau, double* T, int64_t ldt, void* stream);

/* sample_update (randomized.py:107-135): Bnew (ell x n2) = [S12 - S11 R11^{-1}
 * R12; S22] where S (ell x (b + n2)) is the pivoted sample.  *degenerate
 * (host) = 1 when any |R11_jj| < eps^(3/4) frob (Bnew untouched). */
int rq_sample_update(rq_handle_t h, int64_t ell, int64_t b, int64_t n2, const double* S,
                     int64_t lds, const double* R11, const double* R12, int64_t ldr,
                     double frob, double* Bnew, int64_t ldb, int32_t* degenerate,
                     void* stream);

/* qr_blocked (qrcp.py:222-252): in-place unpivoted blocked QR of A (m x n) to
 * rank k; Y (m x k), tau (k).  counters (host, may be NULL) accumulate the
 * OpCounters contribution [gemm, level2, bytes]. */
int rq_qr_blocked(rq_handle_t h, int64_t m, int64_t n, int64_t k, int64_t b, double* A,
                  int64_t lda, double* Y, int64_t ldy, double* tau, int64_t* counters,
                  void* stream);

/* q_columns (qrcp.py:53-60): leading `cols` columns of I - Y T Y^T */
int rq_q_columns(rq_handle_t h, int64_t m, int64_t nref, int64_t cols, const double* Y,
                 int64_t ldy, const double* tau, int64_t b, double* Q, int64_t ldq,
                 void* stream);

/* ||A||_F into a device scalar */
/* column_norms (kernels.py:184-186; qrcp.py:258 qr_presorted): out[j] =
 * ||A[:, j]||_2, bit-identical to np.linalg.norm(A, axis=0) on an F-order
 * array (sequential = 0: numpy's pairwise sum) or a C-order one
 * (sequential = 1: row-order sum).  Device pointers. */
int rq_column_norms(rq_handle_t h, const double* A, int64_t m, int64_t n, int64_t lda,
                    int sequential, double* out, void* stream);
int rq_frob_norm(rq_handle_t h, const double* A, int64_t m, int64_t n, int64_t lda,
                 double* out, void* stream);

/* downdate_norms / NormTracker.downdate (kernels.py:189-192, 225-233):
 * out[j] = sqrt(max(norms[j]^2 - row[j*inc]^2, 0)), bit-identical to numpy;
 * when orig_sq and unsafe are given, unsafe[j] = (out[j]^2 before the root) <
 * guard * orig_sq[j], the columns the caller must recompute exactly.
 * Device pointers; out may alias norms. */
int rq_downdate_norms(rq_handle_t h, const double* norms, const double* row, int64_t inc,
                      int64_t n, const double* orig_sq, double guard, double* out,
                      int32_t* unsafe, void* stream);

/* ---------------------------------------------------------------- host Omega stream */

/* count values of numpy's Philox(key = k0 + 2^64 k1).standard_normal() stream,
 * starting at raw 64-bit draw `raw` (0 = a fresh RngState), written to out;
 * *raw_end = raw position of the next value.  Bit-identical to numpy (its own
 * ziggurat decoder, libnpyrandom.a), decoded by `threads` host threads.
 * Replaces the draw loop of the reference's RngState (pkg/src/rqrcp/rng.py:16-41). */
int rq_omega_fill(uint64_t k0, uint64_t k1, uint64_t raw, double* out, int64_t count, int threads,
                  uint64_t* raw_end);

/* ---------------------------------------------------------------- instrumentation */

/* tuning knobs: "force_select" / "force_panel" (0 = size heuristic, 1 = grid
 * cooperative variant, 2 = single-cluster variant), "select_cluster_max_cols",
 * "panel_cluster_max_rows" (size thresholds of the heuristic), "fast_panel"
 * (1 = CholeskyQR2 + Householder-reconstruction panel first, falling back to
 * the column-by-column kernel when the panel is ill-conditioned; 0 = always
 * column-by-column), "fast_panel_max_ctas", "fast_panel_spec", "use_rank_update",
 * "select_reg", "select_fused" (grid select: barrier counter and key slot in
 * one 16-byte word), "select_max_ctas", "overlap_select", "overlap_sel_ctas"
 * (next block's select beside the trailing update), "sel_cpg2_cols" (that
 * select takes two columns per 8-lane group from this sample width down),
 * "select_on_main" / "select_main_mflop" (the select goes on the main stream
 * once the trailing update is below this many MFLOP), "su_gemm",
 * "overlap_inner", "overlap_panel_ctas" (inner product beside the fast panel),
 * "block_finish" (X, R12 and the sample update fused per column tile),
 * "sel_balance" (x 1e-6: SM share of a shared-memory select beside the
 * trailing update, from the trailing rows), "use_tc" / "tc_tma" / "tc_variant"
 * / "tc_splits" (plain products: DMMA GEMM family, TMA feed, tile family and
 * split-K overrides), "ru_tma" / "ru_big" (trailing update variants),
 * "inner_kernel" / "inner_ktiles", "fast_panel_pad", "omega_ahead",
 * "floor_lookahead", "t_inverse", "panel_halves", "degen_commit",
 * "finish_narrow", "inner32", "panel_rows_per_cta", "profile_trace",
 * "debug_timers"; unknown names return RQ_ERR_INVALID */
int rq_set_option(rq_handle_t h, const char* name, int64_t value);

/* debug: phase timers written by the kernels when "debug_timers" is set */
int rq_debug_read(rq_handle_t h, int64_t* out, int n);

/* total kernel launches issued by this library since load (all handles) */
int64_t rq_launch_count(void);

/* kernel families timed by the profiler (CUDA events around each launch on
 * its own stream); index order of rq_profile_read's arrays */
#define RQ_PROF_SKETCH 0
#define RQ_PROF_INNER 1
#define RQ_PROF_UPDATE 2
#define RQ_PROF_SMALL_GEMM 3
#define RQ_PROF_SELECT 4
#define RQ_PROF_PANEL 5
#define RQ_PROF_SAMPLE_UPDATE 6
#define RQ_PROF_SWAP 7
#define RQ_PROF_MISC 8
#define RQ_PROF_LIB_GEMM 9   /* cuBLAS DGEMM for plain scratch products (not this library's kernels) */
#define RQ_PROF_NUM 10

int rq_profile_enable(rq_handle_t h, int on);
int rq_profile_reset(rq_handle_t h);
/* synchronises pending events; each array has RQ_PROF_NUM entries: launches,
 * summed kernel milliseconds, algorithmic flops and algorithmic bytes */
int rq_profile_read(rq_handle_t h, int64_t* launches, double* ms, double* flops, double* bytes);

/* launch trace of the profiled launches since the last rq_profile_reset (set
 * option "profile_trace" first): family index, start and end in ms on the
 * device timeline; writes min(cap, count) records and the total in *count */
int rq_profile_trace(rq_handle_t h, int64_t cap, int32_t* cat, double* start_ms, double* end_ms,
                     int64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* RQRCP_B200_H */
