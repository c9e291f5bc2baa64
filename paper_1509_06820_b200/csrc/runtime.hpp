// Host runtime for the sm_100a RQRCP library: device handle, grow-only
// workspace arena, error plumbing and the launch helpers shared by the
// drivers (driver.cu) and the C-ABI (abi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace rq {

struct CudaError : std::runtime_error {
  int code;
  CudaError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RQ_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      throw ::rq::CudaError(-3, std::string(#expr) + ": " + cudaGetErrorString(_e) +   \
                                    " (" + __FILE__ + ":" + std::to_string(__LINE__) + \
                                    ")");                                              \
  } while (0)

#define RQ_CHECK_LAUNCH() RQ_CUDA(cudaGetLastError())

struct InvalidArg : std::runtime_error {
  explicit InvalidArg(const std::string& m) : std::runtime_error(m) {}
};

// Kernel families timed by the optional in-driver profiler (bench.py reads
// them through rq_profile_*): CUDA events bracket every launch of a family on
// the stream it runs on.
enum ProfCat {
  kProfSketch = 0,   // B = Omega A (initial + resamples)
  kProfInner,        // G = Y^T C (stage 1, split-K)
  kProfUpdate,       // C -= Y X (stage 2/3: R12 rows + trailing update)
  kProfSmallGemm,    // X = T^T G, TRQRCP/TUXV side products, Q formation
  kProfSelect,       // pivot selection (cooperative)
  kProfPanel,        // panel QR + T (cooperative)
  kProfSampleUpd,    // sample update
  kProfSwap,         // swap replay
  kProfMisc,         // copies, norms, fills
  kProfNum
};
struct ProfStat {
  int64_t launches = 0;
  double ms = 0.0, flops = 0.0, bytes = 0.0;
};

// cudaFuncSetAttribute memoised per (kernel, device, attribute): kernel
// attributes are per device, and one process may drive several GPUs (one
// handle each).  Dynamic shared memory is only ever raised.
void kernel_attr(const void* func, cudaFuncAttribute attr, int value);

// total kernel launches issued by the library (all handles)
void count_launch(int n = 1);
int64_t launch_count();

class Handle;
// RAII timing scope (no-op unless profiling is enabled on the handle)
class ProfScope {
 public:
  ProfScope(Handle& h, int cat, double flops, double bytes, cudaStream_t s);
  ~ProfScope();

 private:
  Handle* h_;
  int idx_ = -1;
  cudaStream_t s_;
};

class Handle {
 public:
  explicit Handle(int device);
  ~Handle();
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  // grow-only named device buffer; synchronises `s` before re-allocating
  void* buf(const std::string& name, size_t bytes, cudaStream_t s);
  void* host_pinned(const std::string& name, size_t bytes, cudaStream_t s);
  // side stream + fork/join events for the select || trailing-update overlap,
  // and the speculative driver's retire events (created once per handle)
  cudaStream_t side_stream();
  cudaStream_t copy_stream();
  // the speculative driver's per-block abort-word snapshots (4-byte D2H copies)
  // go through their own stream: on the compute stream each one is ~10 us of
  // copy-engine latency between two blocks
  cudaStream_t stat_stream();
  cudaEvent_t ev_stat = nullptr;
  cudaStream_t omega_stream();   // uploads of pre-drawn resample Omega
  cudaEvent_t ev_copy = nullptr;
  cudaEvent_t ev_omega = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<cudaEvent_t> ring_ev;

  // kernel-variant overrides (0 = size heuristic, 1 = grid, 2 = cluster)
  int force_select = 0, force_panel = 0;
  // size heuristics: cluster variant when the work per step is small enough
  // (crossovers measured on B200: tools/variant_sweep.py, profiles/r01_variant_sweep.jsonl)
  int64_t select_cluster_max_cols = 1024;   // nt threshold
  int64_t panel_cluster_max_rows = 3072;    // mm threshold (bw <= 64 only)
  int64_t panel_rows_per_cta = 128;         // cluster variant: rows per CTA (power-of-2 CTA count)
  int select_max_ctas = 0;                  // cap of the grid variant (0 = one CTA per SM)
  bool select_reg = true;                   // register-resident select (v5) where it fits
  bool select_fused = true;                 // v5 grid variant: barrier counter and key in one 16-byte word
  bool omega_ahead = true;                  // pre-draw resample Omega on a host thread
  int floor_lookahead = 1;                  // speculative blocks queued once near the noise floor
  bool t_inverse = true;                    // T factor as a DMMA triangular inverse (nb <= 64)
  bool panel_halves = true;                 // 65..128-wide speculative panels as two fast halves
  bool degen_commit = true;                 // fast panel commits clearly degenerate R11 (block_finish resamples)
  bool finish_narrow = true;                // block_finish: 32-column tiles when 64 would leave SMs idle
  bool use_tc = true;                       // plain GEMMs through tc_gemm (tc_gemm.cu)
  int tc_variant = -1;                      // tc_gemm tile family override (-1 = by shape)
  int tc_splits = 0;                        // tc_gemm split-K override (0 = by shape)
  bool tc_tma = true;                       // tc_gemm operands through TMA (tc_tma.cuh; 16-byte aligned operands)

  bool use_rank_update = true;
  bool fast_panel = true;   // CholeskyQR2 + Householder reconstruction panel (panel_fast.cu)
  int fast_panel_max_ctas = 0;  // 0 = one CTA per SM
  int fast_panel_pad = 4;       // smem row stride of the fast panel: n8 + pad doubles (4: the
                                // DMMA fragment loads of a 16-lane phase hit 16 distinct banks)
  // speculative driver on a declined fast panel: 0 = always rewind, 1 = rewind
  // once then queue the exact kernel behind every fast panel, 2 = never rewind
  int fast_panel_spec = 1;
  // speculative RQRCP: next block's select concurrently with the trailing update
  bool overlap_select = true;
  bool su_gemm = true;        // sample update as M = S11 R11^-1 then a rank-b GEMM
  // inner GEMM's P_below^T C_below part concurrently with the fast panel
  bool overlap_inner = true;
  int overlap_panel_ctas = 0;   // SMs for the fast panel while it overlaps (0 = size rule)
  // ... then X, R12 and the sample update fused per column tile (csrc/finish.cu)
  bool block_finish = true;
  bool ru_two_ctas = false;  // rank update: two single-buffered CTAs per SM
  int ru_skew_ns = 0;
  bool ru_big = true;        // rank update: 128 x 64 tiles, C through registers
  int ru_tma = 2;            // rank update: the TMA-fed kernel (rank_update_tma.cu) where it applies;
                             // 0 off, 1 C from HBM in the epilogue, 2/3 C tile prefetched by TMA
  bool inner_kernel = true;  // H = P^T C: tall-skinny split-K kernel (csrc/inner.cu)
  int inner_ktiles = 16;     // ... k-tiles (32 deep) per CTA
  bool inner32 = true;       // ... also for 32-row blocks (b = 32)
  int64_t sel_cpg2_cols = 6400; // overlapped v5 select: 2 columns per group at or below this sample width
  bool select_on_main = true;    // overlapped select on the main stream once it outlasts the update
  int select_main_mflop = 5000;  // ... i.e. below this much trailing-update work (MFLOP)
  int overlap_sel_ctas = 0;   // SMs for the overlapped select (0 = size heuristic)
  int sel_balance = 200;      // v4 select/update balance constant (x 1e-6, overlap_split; cfg5 sweeps: profiles/r02_cfg5_sel_balance.jsonl)
  bool gemm_vec16 = true;
  long long* dbg = nullptr;  // optional device phase-timer buffer (debug)

  // profiler
  bool profiling = false;
  ProfStat stats[kProfNum];
  // optional launch trace (family, start, end in ms from the last reset)
  struct TraceRec {
    int cat;
    double start_ms, end_ms;
  };
  bool tracing = false;
  std::vector<TraceRec> trace;
  int prof_begin(int cat, double flops, double bytes, cudaStream_t s);
  void prof_end(int idx, cudaStream_t s);
  void prof_collect();  // synchronises the pending events into `stats`
  void prof_reset();

 private:
  struct PendEv {
    int cat;
    double flops, bytes;
    cudaEvent_t a, b;
  };
  std::vector<PendEv> pend_;
  cudaEvent_t trace_base_ = nullptr;
  cudaStream_t side_ = nullptr;
  cudaStream_t copy_ = nullptr;
  cudaStream_t stat_ = nullptr;
  cudaStream_t omega_ = nullptr;
  std::vector<cudaEvent_t> free_ev_;
  cudaEvent_t take_event();
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    bool pinned = false;
  };
  std::map<std::string, Buf> bufs_;
};

// ------------------------------------------------------------------ GEMM
// C = alpha * op(A) op(B) + beta * C on `s` (gemm.cu).  Column-major.
void gemm(Handle& h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
          const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
          int64_t ldc, cudaStream_t s, const Status* st = nullptr, int cat = kProfSmallGemm);

// second-generation DMMA GEMM (tc_gemm.cu); false when disabled or op(A) and
// op(B) are both transposed (the caller then uses gemm_f64_kernel)
bool tc_gemm(Handle& h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
             const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
             int64_t ldc, cudaStream_t s, const Status* st, int cat);

// TMA-fed persistent C -= Y X for K in {32, 64} (rank_update_tma.cu); false if
// not applicable (option ru_tma off, shape, alignment)
bool rank_update_tma(Handle& h, int64_t M, int64_t N, int64_t K, const double* Y, int64_t ldy,
                     const double* X, int64_t ldx, double* C, int64_t ldc, cudaStream_t s,
                     const Status* st, int cat, int max_ctas, Status* snap);

// persistent C -= Y X for K <= 64 (rank_update.cu); false if not applicable
bool rank_update(Handle& h, int64_t M, int64_t N, int64_t K, const double* Y, int64_t ldy,
                 const double* X, int64_t ldx, double* C, int64_t ldc, cudaStream_t s,
                 const Status* st, int cat, int max_ctas = 0, Status* snap = nullptr,
                 const double* Csrc = nullptr, int64_t ldcs = 0, int extra_rows = 0);

// ------------------------------------------------------------------ kernels (small.cu, select.cu, panel.cu)
struct SelectOut {
  double* S; int64_t lds;     // pivoted transformed sample (ell x nt)
  int64_t* piv;               // want entries: step j swapped (j, piv[j])
  double* Ys; int64_t ldys;   // optional sample reflectors (ell x want)
  double* taus;               // optional
};
// b greedy steps of pivoted QR on the ell x nt sample (randomized.py:85-104).
// abort_on_short: set Status.abort = kAbortShortSample when got < want.
void select_pivots(Handle& h, int64_t ell, int64_t nt, int64_t want, const double* B,
                   int64_t ldb, const SelectOut& out, Status* st, bool abort_on_short,
                   int64_t i0, cudaStream_t s, int max_ctas = 0);

struct PanelOut {
  double* Rdst; int64_t ldr; int64_t rrows;   // transformed panel rows [0, rrows)
  double* Y; int64_t ldy;                      // unit lower reflectors (mm x bw)
  double* tau;
  double* T; int64_t ldt;                      // optional T factor of the committed columns
};
// kPanelCommitIfFull: commit only when every column is usable (otherwise the
// driver resamples; with raise_abort the kernel also sets Status.abort)
enum PanelPolicy { kPanelCommitIfFull = 0, kPanelCommitUsable = 1, kPanelCommitAll = 2 };
// Householder QR of an mm x bw panel (qrcp.py:206-219) + _panel_rank
// (randomized.py:150-155) + build_t_matrix (kernels.py:139-147).
// allow_fast: try panel_fast first.  With raise_abort && fast_aborts
// (speculative driver) the fast path runs alone and a decline aborts the
// block (kAbortPanelFast); otherwise the exact kernel follows it on the
// stream and runs only if the fast path declined.
void panel_qr(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
              const PanelOut& out, double tol, PanelPolicy policy, bool raise_abort, Status* st,
              int64_t i0, cudaStream_t s, bool allow_fast = true, bool fast_aborts = true);

// CholeskyQR2 + Householder reconstruction of the same panel (panel_fast.cu).
// Returns the device flag the exact kernel checks (1 = committed, 0 = the
// exact kernel must run), or nullptr when the panel shape is not eligible.
// abort_on_decline (speculative driver): a declined panel sets Status.abort =
// kAbortPanelFast at block i0 instead of leaving the work to the exact kernel.
bool panel_fast_eligible(const Handle& h, int64_t mm, int64_t bw);
// max_ctas caps the grid (0: one CTA per SM); defer_zero leaves the panel rows
// below the diagonal unzeroed (the caller zeroes them later); m_rowmajor / m_ld
// receive the committed M (Y_below = P_below M) as a row-major ld x ld block.
const int* panel_fast(Handle& h, int64_t mm, int64_t bw, const double* P, int64_t ldp,
                      const PanelOut& out, double tol, Status* st, cudaStream_t s,
                      bool abort_on_decline = false, int64_t i0 = 0, int max_ctas = 0,
                      bool defer_zero = false, const double** m_rowmajor = nullptr,
                      int64_t* m_ld = nullptr, const double* S11 = nullptr,
                      int64_t lds11 = 0, double* msu = nullptr, double* a12 = nullptr,
                      int64_t l2_extra = 0, int usable_total = 0, bool degen_commit = false);

// Rest of a speculative RQRCP block after a committed fast panel, one CTA per
// 64-column tile of the trailing matrix (csrc/finish.cu):
//   X = A1^T C_top + A2^T H, R12 = C_top - Y_top X (in place),
//   B_new = [S12 - Msu R12; S22], panel rows below the diagonal zeroed,
//   and the abort-word snapshot for the deferred trailing update.
struct FinishArgs {
  int64_t nt2, mm; int b, ell;
  double* Ctop; int64_t ldw;        // work rows [i0, i0+b) x cols [i0+b, n): C_top in, R12 out
  const double* H;                  // b x nt2, ld b
  const double* A12;                // [A1; A2], b x b row-major each
  const double* Ytop; int64_t ldy;  // b x b unit lower
  const double* Msu;                // b x b
  const double* S; int64_t lds;     // sample columns [b, b+nt2): S12 rows < b, S22 rows >= b
  double* X;                        // b x nt2, ld b
  double* Bn; int64_t ldb;          // ell x nt2
  double* Pz;                       // panel rows below the diagonal: (mm - b) x b, ld ldw
  Status* st; Status* pre;
  // optional: the fast panel committed a clearly degenerate R11 (Status.degenerate):
  // the last CTA to finish raises kAbortDegenerate at block i0 (after block 0's
  // snapshot in `pre`, so the trailing update still runs)
  unsigned int* done_ctr;
  int64_t i0;
};
bool block_finish(Handle& h, const FinishArgs& f, cudaStream_t s);

// H (64 x N, ld ldh) = P^T C with P (K x 64) and C (K x N) column-major,
// on at most max_ctas SMs (csrc/inner.cu); false when the shape does not qualify

bool inner_gemm(Handle& h, int64_t M, int64_t N, int64_t K, const double* P, int64_t ldp,
                const double* C, int64_t ldc, double* H, int64_t ldh, cudaStream_t s,
                const Status* st, int max_ctas, int cat);

// B_new = [S12 - M R12; S22] with M = S11 R11^{-1} already formed (by the
// fast panel of the same block, which also cleared the degenerate guard).
void sample_update_pre(Handle& h, int64_t ell, int64_t b, int64_t n2, const double* S,
                       int64_t lds, const double* M, const double* R12, int64_t ldr,
                       double* Bnew, int64_t ldb, Status* st, cudaStream_t s);

// B_new = [S12 - S11 R11^{-1} R12; S22] (randomized.py:107-135).  Writes
// Status.degenerate; with abort_on_degenerate also sets Status.abort.
void sample_update(Handle& h, int64_t ell, int64_t b, int64_t n2, const double* S, int64_t lds,
                   const double* R11, const double* R12, int64_t ldr, double frob,
                   double* Bnew, int64_t ldb, Status* st, bool abort_on_degenerate, int64_t i0,
                   cudaStream_t s);

// replay the select swaps at offset i0 on work columns, perm, swap log and
// row followers (randomized.py:138-147)
struct SwapTargets {
  double* work; int64_t ldw; int64_t m;
  int64_t* perm;
  int64_t* log; int64_t log_cap;
  double* Wf; int64_t ldwf; int64_t wf_cols;   // optional W rows (TRQRCP)
  double* Rf; int64_t ldrf; int64_t rf_rows;   // optional R columns (TRQRCP)
};
void apply_swaps(Handle& h, const int64_t* piv, int64_t got_max, int64_t i0,
                 const SwapTargets& t, Status* st, cudaStream_t s);

// misc
// np.linalg.norm(A, axis=0) bit for bit (pairwise per column, or sequential
// in row order when mirroring a C-order host array)
void column_norms(Handle& h, const double* A, int64_t m, int64_t n, int64_t lda, bool sequential,
                  double* out, cudaStream_t s);
void frob_norm(Handle& h, const double* A, int64_t m, int64_t n, int64_t lda, double* out,
               cudaStream_t s);
void copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
            int64_t cols, cudaStream_t s, const Status* st = nullptr);
// sqrt(max(norms^2 - row^2, 0)) elementwise, optional recompute flags (small.cu)
void downdate_norms(const double* norms, const double* row, int64_t inc, int64_t n,
                    const double* orig_sq, double guard, double* out, int32_t* unsafe,
                    cudaStream_t s);
// snapshot (restore = false) / conditional restore of a two-half panel's
// columns, reflectors and level-2 counters (small.cu halves_guard_kernel)
void halves_guard(Handle& h, double* work, int64_t ldw, int64_t mm, int64_t cols, Status* st,
                  bool restore, int64_t i0, double* Y, int64_t ldy, double* tau, cudaStream_t s);
void fill2d(double* dst, int64_t ldd, int64_t rows, int64_t cols, double v, cudaStream_t s,
            const Status* st = nullptr);
void transpose(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
               int64_t cols, cudaStream_t s);
void scatter_cols(const double* src, int64_t lds, const int64_t* perm, double* dst,
                  int64_t ldd, int64_t rows, int64_t cols, cudaStream_t s);
void set_identity(double* dst, int64_t ldd, int64_t rows, int64_t cols, cudaStream_t s);
// full T factor of Y (mm x nb) from its Gram matrix (kernels.py:139-147)
void t_factor(Handle& h, const double* Y, int64_t ldy, int64_t mm, int64_t nb,
              const double* tau, double* T, int64_t ldt, cudaStream_t s,
              const Status* st = nullptr);

}  // namespace rq
