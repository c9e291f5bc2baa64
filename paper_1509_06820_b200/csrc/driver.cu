// Native block-loop drivers for RQRCP / RSRQRCP / SSRQRCP / TRQRCP and the
// unpivoted pieces TUXV needs (qr_blocked, q_columns).
//
// Control flow follows randomized.py:183-266 (_randomized_factor) and
// truncated.py:70-174 (trqrcp) exactly, including the three resample
// triggers.  The GPU does not wait for the host between blocks: blocks are
// enqueued speculatively (up to kLookahead ahead) under the assumption that no
// trigger fires.  Each trigger is detected on the device by the kernel that
// evaluates it (select: got < want; panel: usable < got; sample update:
// degenerate R11), which records the stage and block in Status and sets
// Status.abort -- every later kernel in the queue then returns immediately.
// The host notices the flag when it retires the oldest speculative block,
// rewinds to the failing block and replays the reference's branch
// synchronously (resample from the host Omega stream, retry), then resumes
// speculation.  Since a failing stage never commits anything the reference
// would not have committed, the device state at the abort point equals the
// reference's state at that branch.
#include <cstring>
#include <deque>
#include <thread>
#include <vector>

#include "driver.hpp"

extern "C" int rq_omega_fill(uint64_t k0, uint64_t k1, uint64_t raw, double* out, int64_t count,
                             int threads, uint64_t* raw_end);

namespace rq {

namespace {

constexpr int kLookahead = 3;

struct Pending {
  int64_t i0, bw;
  Counters stage, update;
  bool has_update;
  int slot;
};

class Factor {
 public:
  Factor(Handle& h, const FactorParams& p) : h_(h), p_(p), s_(p.stream), ev_(h.ring_ev) {}
  ~Factor() {
    if (ahead_.joinable()) ahead_.join();
  }

  FactorResult run();

 private:
  Handle& h_;
  const FactorParams& p_;
  cudaStream_t s_;
  Status* st_ = nullptr;   // device
  Status* hst_ = nullptr;  // pinned
  Status* pre_ = nullptr;  // device: abort word before a block's sample update
  int* hring_ = nullptr;   // pinned abort snapshots
  std::vector<cudaEvent_t>& ev_;   // retire events (owned by the handle)
  double *B_ = nullptr, *S_ = nullptr, *T_ = nullptr, *G_ = nullptr, *X_ = nullptr;
  double *om_d_ = nullptr, *om_h_ = nullptr, *P_ = nullptr, *Z_ = nullptr;
  int64_t* piv_ = nullptr;
  double frob_ = 0.0, tol_ = 0.0;
  // a declined speculative fast panel rewinds the lookahead; after the first
  // one (declines cluster near the noise floor) the exact kernel is queued
  // behind every fast panel instead
  bool fast_aborts_ = true;
  // set once a block hit the noise floor (a degenerate or panel-rank trigger,
  // or a declined fast panel): the synchronous path then goes straight to the
  // exact panel, whose verdict the fast one would only have declined to give
  bool near_floor_ = false;
  bool floor_seen_ = false;            // any noise-floor trigger: one block of lookahead
  unsigned int* fin_done_ = nullptr;   // block_finish's CTA counter (degenerate verdict)
  Counters c_;
  int64_t m_ = 0, n_ = 0, k_ = 0, b_ = 0, ell_ = 0;

  // Resample Omega look-ahead: the stream is sequential, so the next l*m
  // draws (the most one resample can take) are drawn on a host thread and
  // uploaded while the factorization runs; a resample then takes its draws
  // from the device copy instead of waiting for the host generator.
  std::thread ahead_;
  double *ah_h_ = nullptr, *ah_d_ = nullptr;
  int64_t ah_n_ = 0, ah_pos_ = 0;
  int ah_rc_ = 0;
  void start_ahead(bool after_event);
  uint64_t om_raw_ = 0;   // native stream: raw Philox counter after the draws so far
  bool has_omega() const { return p_.omega_native || p_.omega_fn != nullptr; }
  // the next `count` draws of the Omega stream into host memory
  int draw_host(int64_t count, double* dst) {
    if (p_.omega_native) {
      uint64_t end = 0;
      const int rc = rq_omega_fill(p_.omega_k0, p_.omega_k1, om_raw_, dst, count,
                                   std::max(1, p_.omega_threads), &end);
      if (rc == 0) om_raw_ = end;
      return rc;
    }
    return p_.omega_fn(p_.omega_user, 1, count, dst);
  }
  const double* omega_take(int64_t rows, int64_t cols);

  void sync() { RQ_CUDA(cudaStreamSynchronize(s_)); }
  Status read_status() {
    RQ_CUDA(cudaMemcpyAsync(hst_, st_, sizeof(Status), cudaMemcpyDeviceToHost, s_));
    sync();
    return *hst_;
  }
  void touch(Counters& c, int64_t elems) { c.bytes_touched += 8 * elems; }

  void draw_omega(int64_t rows, int64_t cols);
  void first_sample();
  void fresh_sample(int64_t i0);
  void select(int64_t i0, int64_t want, bool spec, cudaStream_t s = nullptr, int max_ctas = 0);
  void swaps(int64_t i0, int64_t got);
  void panel(int64_t i0, int64_t got, PanelPolicy pol, bool spec, Counters& c,
             bool allow_fast = true);
  void stages(int64_t i0, int64_t bw, Counters& c, bool defer_trailing = false,
              bool g_ready = false);
  bool panel_overlap_inner(int64_t i0, int64_t bw);
  bool panel_halves(int64_t i0, int64_t got);
  bool msu_ready_ = false;   // the fast panel left the sample update's M in "su_Mpre"
  bool fin_ready_ = false;   // ... and A1 = Y1 T, A2 = M T in "fin_A12": block_finish() path
  void trailing(int64_t i0, int64_t bw, int max_ctas, const Status* pred, cudaStream_t s = nullptr);
  void stream_out(int64_t upto, bool final);
  int64_t host_done_ = 0;   // columns whose host copies are enqueued
  int overlap_split(int64_t i0, int64_t bw) const;
  bool select_is_longer(int64_t i0, int64_t bw) const;
  int panel_split(int64_t mm, int64_t nt2, int64_t bw) const;
  void update(int64_t i0_new, int64_t bw, bool spec, Counters& c);
  bool slow_block(int64_t& i0, bool resampled, int64_t& rank, bool resume_panel = false);
};

void Factor::draw_omega(int64_t rows, int64_t cols) {
  if (!has_omega()) throw InvalidArg("no Omega source for a (re)sample");
  // the pinned staging buffer is reused: every caller has synchronised the
  // stream, so no earlier H2D copy is still reading it
  const int rc = draw_host(rows * cols, om_h_);
  if (rc != 0) throw InvalidArg("Omega callback failed");
  RQ_CUDA(cudaMemcpyAsync(om_d_, om_h_, (size_t)rows * cols * 8, cudaMemcpyHostToDevice, s_));
}

// after_event: the device copy is still being read by work enqueued on s_
// (h_.ev_omega recorded there), so the upload waits for it
void Factor::start_ahead(bool after_event) {
  // the look-ahead thread draws natively only: a callback into the caller
  // (Python) from a second thread could wait on the caller's lock
  if (!p_.omega_native || !h_.omega_ahead) return;
  const int64_t n = ell_ * m_;
  ah_h_ = (double*)h_.host_pinned("omega_ahead_h", (size_t)n * 8, s_);
  ah_d_ = (double*)h_.buf("omega_ahead_d", (size_t)n * 8, s_);
  ah_n_ = n;
  ah_pos_ = 0;
  ah_rc_ = 0;
  cudaStream_t os = h_.omega_stream();
  if (after_event) RQ_CUDA(cudaEventRecord(h_.ev_omega, s_));
  const int dev = h_.device;
  ahead_ = std::thread([this, n, os, dev, after_event] {
    cudaSetDevice(dev);
    ah_rc_ = draw_host(n, ah_h_);
    if (ah_rc_ != 0) return;
    if (after_event) cudaStreamWaitEvent(os, h_.ev_omega, 0);
    if (cudaMemcpyAsync(ah_d_, ah_h_, (size_t)n * 8, cudaMemcpyHostToDevice, os) != cudaSuccess ||
        cudaStreamSynchronize(os) != cudaSuccess)
      ah_rc_ = 1;
  });
}

// The next rows*cols draws of the Omega stream as a device pointer ordered on
// s_: pre-drawn ones first, the rest drawn now (stream order preserved), then
// a new look-ahead batch.
const double* Factor::omega_take(int64_t rows, int64_t cols) {
  const int64_t need = rows * cols;
  if (!ahead_.joinable() && ah_n_ == 0) {
    draw_omega(rows, cols);
    return om_d_;
  }
  if (ahead_.joinable()) ahead_.join();
  if (ah_rc_ != 0) throw InvalidArg("Omega callback failed");
  const int64_t have = ah_n_ - ah_pos_;
  if (need < have) {
    const double* p = ah_d_ + ah_pos_;
    ah_pos_ += need;
    return p;
  }
  // the rest of the batch, then fresh draws behind it
  if (have > 0)
    RQ_CUDA(cudaMemcpyAsync(om_d_, ah_d_ + ah_pos_, (size_t)have * 8, cudaMemcpyDeviceToDevice, s_));
  if (need > have) {
    const int rc = draw_host(need - have, om_h_);
    if (rc != 0) throw InvalidArg("Omega callback failed");
    RQ_CUDA(cudaMemcpyAsync(om_d_ + have, om_h_, (size_t)(need - have) * 8, cudaMemcpyHostToDevice,
                            s_));
  }
  ah_n_ = 0;
  start_ahead(true);
  return om_d_;
}

// make_sample(work, ell, rng) (randomized.py:69-82; truncated.py:97)
void Factor::first_sample() {
  const double* om = p_.omega0;
  if (om == nullptr) {
    draw_omega(ell_, m_);
    om = om_d_;
  }
  // the sketch is a plain GEMM outside the speculative chain (tc_gemm.cu)
  gemm(h_, false, false, ell_, n_, m_, 1.0, om, ell_, p_.work, p_.ldw, 0.0, B_, ell_, s_, nullptr,
       kProfSketch);
  c_.gemm_flops += 2 * ell_ * m_ * n_;
  touch(c_, ell_ * m_ + m_ * n_ + ell_ * n_);
}

// fresh_sample(i0) (randomized.py:199-202) / _sketched_sample (truncated.py:53-67)
void Factor::fresh_sample(int64_t i0) {
  sync();
  const int64_t mm = m_ - i0, nt = n_ - i0;
  const double* om = omega_take(ell_, mm);
  const double* At = p_.work + i0 + i0 * p_.ldw;
  gemm(h_, false, false, ell_, nt, mm, 1.0, om, ell_, At, p_.ldw, 0.0, B_, ell_, s_, nullptr,
       kProfSketch);
  c_.gemm_flops += 2 * ell_ * mm * nt;
  touch(c_, ell_ * mm + mm * nt + ell_ * nt);
  if (p_.truncated && i0) {
    // B -= (Omega Y[i0:, :i0]) W[i0:, :i0]^T
    gemm(h_, false, false, ell_, i0, mm, 1.0, om, ell_, p_.Y + i0, p_.ldy, 0.0, Z_, ell_, s_,
         nullptr, kProfSketch);
    gemm(h_, false, true, ell_, nt, i0, -1.0, Z_, ell_, p_.W + i0, p_.ldW, 1.0, B_, ell_, s_,
         nullptr, kProfSketch);
    c_.gemm_flops += 2 * ell_ * mm * i0 + 2 * ell_ * i0 * nt;
    touch(c_, mm * i0 + nt * i0);
  }
}

void Factor::select(int64_t i0, int64_t want, bool spec, cudaStream_t s, int max_ctas) {
  SelectOut o{S_, ell_, piv_, nullptr, 0, nullptr};
  select_pivots(h_, ell_, n_ - i0, want, B_, ell_, o, st_, spec, i0, s ? s : s_, max_ctas);
}

void Factor::swaps(int64_t i0, int64_t got) {
  SwapTargets t{};
  t.work = p_.work; t.ldw = p_.ldw; t.m = m_;
  t.perm = p_.perm; t.log = p_.swaps; t.log_cap = p_.swap_cap;
  if (p_.truncated) {
    t.Wf = p_.W; t.ldwf = p_.ldW; t.wf_cols = k_;
    t.Rf = p_.R; t.ldrf = p_.ldR; t.rf_rows = k_;
  }
  apply_swaps(h_, piv_, got, i0, t, st_, s_);
}

// A 65..128-column speculative panel as two fast 64-column halves (the
// recursive panel QR): Householder QR is column-sequential, so the first 64
// reflectors come from the first 64 columns alone; they are applied to the
// other columns (G = Y1^T P2, P2 -= Y1 T1^T G), whose rows below 64 are then
// factored, and T = [[T1, -T1 (Y1^T Y2) T2], [0, T2]].  Each half commits
// only under the fast panel's margins (else Status.abort rewinds the block
// to the exact kernel), so a commit means every |R_jj| cleared _panel_rank.
bool Factor::panel_halves(int64_t i0, int64_t got) {
  const int64_t mm = m_ - i0, h2 = got - 64;
  if (p_.truncated || got <= 64 || got > 128 || mm < got + 64 || !h_.panel_halves ||
      !panel_fast_eligible(h_, mm, 64) || !panel_fast_eligible(h_, mm - 64, h2))
    return false;
  double* P1 = p_.work + i0 + i0 * p_.ldw;
  double* P2 = P1 + 64 * p_.ldw;
  double* Y1 = p_.Y + i0 + i0 * p_.ldy;
  double* Y2 = Y1 + 64 + 64 * p_.ldy;
  double* G = (double*)h_.buf("ph_G", (size_t)64 * 128 * 8, s_);
  double* X = G + 64 * 64;
  // the first half commits in place; keep the selected columns so a decline
  // of the second half rewinds to them (restored below, on the device)
  halves_guard(h_, P1, p_.ldw, mm, got, st_, false, i0, Y1, p_.ldy, p_.tau + i0, s_);
  PanelOut o1{};
  o1.Y = Y1; o1.ldy = p_.ldy; o1.tau = p_.tau + i0;
  o1.T = T_; o1.ldt = b_;
  o1.Rdst = P1; o1.ldr = p_.ldw; o1.rrows = mm;
  panel_fast(h_, mm, 64, P1, p_.ldw, o1, tol_, st_, s_, true, i0);
  // P2 <- H_64 ... H_1 P2 = P2 - Y1 (T1^T (Y1^T P2))
  if (!inner_gemm(h_, 64, h2, mm, Y1, p_.ldy, P2, p_.ldw, G, 64, s_, st_, 0, kProfPanel))
    gemm(h_, true, false, 64, h2, mm, 1.0, Y1, p_.ldy, P2, p_.ldw, 0.0, G, 64, s_, st_,
         kProfPanel);
  gemm(h_, true, false, 64, h2, 64, 1.0, T_, b_, G, 64, 0.0, X, 64, s_, st_, kProfPanel);
  if (!rank_update(h_, mm, h2, 64, Y1, p_.ldy, X, 64, P2, p_.ldw, s_, st_, kProfPanel))
    gemm(h_, false, false, mm, h2, 64, -1.0, Y1, p_.ldy, X, 64, 1.0, P2, p_.ldw, s_, st_,
         kProfPanel);
  // rows 64.. of the updated columns; the level-2 count of the reference's
  // column-by-column panel includes reflectors 1..64 applied to them
  int64_t l2x = 0;
  for (int64_t j = 0; j < 64; ++j) l2x += (mm - j) * h2;
  PanelOut o2{};
  o2.Y = Y2; o2.ldy = p_.ldy; o2.tau = p_.tau + i0 + 64;
  o2.T = T_ + 64 + 64 * b_; o2.ldt = b_;
  o2.Rdst = P2 + 64; o2.ldr = p_.ldw; o2.rrows = mm - 64;
  panel_fast(h_, mm - 64, h2, P2 + 64, p_.ldw, o2, tol_, st_, s_, true, i0, 0, false, nullptr,
             nullptr, nullptr, 0, nullptr, nullptr, l2x, (int)got);
  // T12 = -T1 (Y1[64:]^T Y2[64:]) T2, T21 = 0
  if (!inner_gemm(h_, 64, h2, mm - 64, Y1 + 64, p_.ldy, Y2, p_.ldy, G, 64, s_, st_, 0,
                  kProfPanel))
    gemm(h_, true, false, 64, h2, mm - 64, 1.0, Y1 + 64, p_.ldy, Y2, p_.ldy, 0.0, G, 64, s_, st_,
         kProfPanel);
  gemm(h_, false, false, 64, h2, h2, 1.0, G, 64, T_ + 64 + 64 * b_, b_, 0.0, X, 64, s_, st_,
       kProfPanel);
  gemm(h_, false, false, 64, h2, 64, -1.0, T_, b_, X, 64, 0.0, T_ + 64 * b_, b_, s_, st_,
       kProfPanel);
  fill2d(T_ + 64, b_, h2, 64, 0.0, s_, st_);
  halves_guard(h_, P1, p_.ldw, mm, got, st_, true, i0, Y1, p_.ldy, p_.tau + i0, s_);
  return true;
}

void Factor::panel(int64_t i0, int64_t got, PanelPolicy pol, bool spec, Counters& c,
                   bool allow_fast) {
  const int64_t mm = m_ - i0;
  if (spec && allow_fast && fast_aborts_ && panel_halves(i0, got)) return;
  PanelOut o{};
  o.Y = p_.Y + i0 + i0 * p_.ldy; o.ldy = p_.ldy;
  o.tau = p_.tau + i0;
  o.T = T_; o.ldt = b_;
  const double* src;
  int64_t lds;
  if (!p_.truncated) {
    src = p_.work + i0 + i0 * p_.ldw; lds = p_.ldw;
    o.Rdst = p_.work + i0 + i0 * p_.ldw; o.ldr = p_.ldw; o.rrows = mm;
  } else {
    // materialize the selected columns: A[i0:, sel] - Y[i0:, :i0] W[sel, :i0]^T (truncated.py:119-123)
    copy2d(p_.work + i0 + i0 * p_.ldw, p_.ldw, P_, mm, mm, got, s_, st_);
    if (i0) {
      gemm(h_, false, true, mm, got, i0, -1.0, p_.Y + i0, p_.ldy, p_.W + i0, p_.ldW, 1.0, P_, mm,
           s_, st_);
      c.gemm_flops += 2 * mm * i0 * got;
      touch(c, mm * got + mm * i0 + got * i0);
    }
    src = P_; lds = mm;
    o.Rdst = p_.R + i0 + i0 * p_.ldR; o.ldr = p_.ldR; o.rrows = got;
  }
  panel_qr(h_, mm, got, src, lds, o, tol_, pol, spec, st_, i0, s_, allow_fast, fast_aborts_);
}

// _block_stages (randomized.py:158-180) / trqrcp W+R update (truncated.py:453-470)
void Factor::stages(int64_t i0, int64_t bw, Counters& c, bool defer_trailing, bool g_ready) {
  const int64_t mm = m_ - i0, nt2 = n_ - i0 - bw;
  if (nt2 <= 0) return;
  const double* Yb = p_.Y + i0 + i0 * p_.ldy;
  if (!p_.truncated) {
    double* C = p_.work + i0 + (i0 + bw) * p_.ldw;
    if (g_ready && fin_ready_) {
      // X, R12, the sample update, the panel's zero fill and the abort
      // snapshot in one launch (csrc/finish.cu); trailing() does C[b:]
      FinishArgs f{};
      f.nt2 = nt2; f.mm = mm; f.b = (int)bw; f.ell = (int)ell_;
      f.Ctop = C; f.ldw = p_.ldw;
      f.H = (const double*)h_.buf("inner_H", 8, s_);
      f.A12 = (const double*)h_.buf("fin_A12", 8, s_);
      f.Ytop = Yb; f.ldy = p_.ldy;
      f.Msu = (const double*)h_.buf("su_Mpre", 8, s_);
      f.S = S_ + bw * ell_; f.lds = ell_;
      f.X = X_; f.Bn = B_; f.ldb = ell_;
      f.Pz = p_.work + i0 + bw + i0 * p_.ldw;
      f.st = st_; f.pre = pre_;
      f.done_ctr = h_.degen_commit ? fin_done_ : nullptr;
      f.i0 = i0;
      if (!block_finish(h_, f, s_)) throw std::runtime_error("block_finish: unsupported shape");
      c.gemm_flops += 2 * mm * bw * nt2 + bw * bw * nt2 + 2 * bw * bw * nt2;
      touch(c, mm * nt2 + mm * bw + bw * nt2);
      if (p_.update_trailing && i0 + bw < m_) {
        c.gemm_flops += 2 * (mm - bw) * bw * nt2;
        touch(c, (mm - bw) * nt2);
      }
      return;
    }
    if (!g_ready &&   // else panel_overlap_inner() assembled G = Y^T C
        !inner_gemm(h_, bw, nt2, mm, Yb, p_.ldy, C, p_.ldw, G_, bw, s_, st_, 0, kProfInner))
      gemm(h_, true, false, bw, nt2, mm, 1.0, Yb, p_.ldy, C, p_.ldw, 0.0, G_, bw, s_, st_,
           kProfInner);
    gemm(h_, true, false, bw, nt2, bw, 1.0, T_, b_, G_, bw, 0.0, X_, bw, s_, st_);
    c.gemm_flops += 2 * mm * bw * nt2 + bw * bw * nt2;
    const bool trail = p_.update_trailing && i0 + bw < m_;
    // defer_trailing: only R12 = C[:b] - Y[:b] X here (its kernel also
    // snapshots the abort word for trailing(), see there); trailing() does C[b:]
    const int64_t rows = (trail && !defer_trailing) ? mm : bw;
    bool snapped = false;
    if (defer_trailing)
      snapped = rank_update(h_, rows, nt2, bw, Yb, p_.ldy, X_, bw, C, p_.ldw, s_, st_,
                            kProfUpdate, 0, pre_);
    if (!snapped) {
      if (defer_trailing)
        RQ_CUDA(cudaMemcpyAsync(&pre_->abort, &st_->abort, sizeof(int), cudaMemcpyDeviceToDevice,
                                s_));
      gemm(h_, false, false, rows, nt2, bw, -1.0, Yb, p_.ldy, X_, bw, 1.0, C, p_.ldw, s_, st_,
           kProfUpdate);
    }
    c.gemm_flops += 2 * bw * bw * nt2;
    touch(c, mm * nt2 + mm * bw + bw * nt2);
    if (trail) {
      c.gemm_flops += 2 * (mm - bw) * bw * nt2;
      touch(c, (mm - bw) * nt2);
    }
    return;
  }
  // G = Yb^T A[i0:, i0+bw:] - (Yb^T Y[i0:, :i0]) W[i0+bw:, :i0]^T
  if (!inner_gemm(h_, bw, nt2, mm, Yb, p_.ldy, p_.work + i0 + (i0 + bw) * p_.ldw, p_.ldw, G_, bw,
                  s_, st_, 0, kProfInner))
    gemm(h_, true, false, bw, nt2, mm, 1.0, Yb, p_.ldy, p_.work + i0 + (i0 + bw) * p_.ldw, p_.ldw,
         0.0, G_, bw, s_, st_, kProfInner);
  c.gemm_flops += 2 * mm * bw * nt2;
  if (i0) {
    if (!inner_gemm(h_, bw, i0, mm, Yb, p_.ldy, p_.Y + i0, p_.ldy, Z_, bw, s_, st_, 0,
                    kProfSmallGemm))
      gemm(h_, true, false, bw, i0, mm, 1.0, Yb, p_.ldy, p_.Y + i0, p_.ldy, 0.0, Z_, bw, s_, st_);
    gemm(h_, false, true, bw, nt2, i0, -1.0, Z_, bw, p_.W + i0 + bw, p_.ldW, 1.0, G_, bw, s_, st_);
    c.gemm_flops += 2 * mm * bw * i0 + 2 * bw * i0 * nt2;
  }
  // W[i0+bw:, i0:i0+bw] = (T^T G)^T = G^T T
  gemm(h_, true, false, nt2, bw, bw, 1.0, G_, bw, T_, b_, 0.0, p_.W + (i0 + bw) + i0 * p_.ldW,
       p_.ldW, s_, st_);
  c.gemm_flops += bw * bw * nt2;
  // R[i0:i0+bw, i0+bw:] = A[i0:i0+bw, i0+bw:] - Y[i0:i0+bw, :i0+bw] W[i0+bw:, :i0+bw]^T
  double* Rr = p_.R + i0 + (i0 + bw) * p_.ldR;
  copy2d(p_.work + i0 + (i0 + bw) * p_.ldw, p_.ldw, Rr, p_.ldR, bw, nt2, s_, st_);
  gemm(h_, false, true, bw, nt2, i0 + bw, -1.0, p_.Y + i0, p_.ldy, p_.W + i0 + bw, p_.ldW, 1.0,
       Rr, p_.ldR, s_, st_);
  c.gemm_flops += 2 * bw * (i0 + bw) * nt2;
  touch(c, bw * n_ + nt2 * (i0 + bw));
}

// C[b:] -= Y[b:] X of the block at i0 (the rows stages() deferred), on at
// most max_ctas SMs (the rest run the next block's select meanwhile)
// Speculative RQRCP with the fast panel: its Y_below = P_below M, so the
// inner product G = Y^T C splits into Y_top^T C_top + M^T (P_below^T C_below).
// The big term H = P_below^T C_below needs only the panel's INPUT columns, so
// it runs on the side stream while the fast panel (capped CTAs) factors them;
// afterwards G is assembled with two b x b x nt2 products and the panel rows
// below the diagonal (left unzeroed for H) are cleared.  A decline aborts the
// block as usual (nothing was written).  Returns false (nothing launched)
// when the shape does not qualify.
bool Factor::panel_overlap_inner(int64_t i0, int64_t bw) {
  const int64_t mm = m_ - i0, nt2 = n_ - i0 - bw;
  if (p_.truncated || nt2 <= 0 || mm <= bw || !panel_fast_eligible(h_, mm, bw)) return false;
  PanelOut o{};
  o.Y = p_.Y + i0 + i0 * p_.ldy; o.ldy = p_.ldy;
  o.tau = p_.tau + i0;
  o.T = T_; o.ldt = b_;
  o.Rdst = p_.work + i0 + i0 * p_.ldw; o.ldr = p_.ldw; o.rrows = mm;
  double* H = (double*)h_.buf("inner_H", (size_t)b_ * n_ * 8, s_);
  cudaStream_t s2 = h_.side_stream();
  RQ_CUDA(cudaEventRecord(h_.ev_fork, s_));
  RQ_CUDA(cudaStreamWaitEvent(s2, h_.ev_fork, 0));
  const double* Mrm = nullptr;
  int64_t ldm = 0;
  double* msu = (double*)h_.buf("su_Mpre", (size_t)b_ * b_ * 8, s_);
  // block_finish() needs a deferred trailing update (the select overlap) and b in {32, 64}
  fin_ready_ = h_.block_finish && (bw == 32 || bw == 64) && ell_ >= bw && p_.update_trailing &&
               i0 + bw < k_ && h_.overlap_select;
  double* a12 = fin_ready_ ? (double*)h_.buf("fin_A12", (size_t)2 * b_ * b_ * 8, s_) : nullptr;
  const int qp = panel_split(mm, nt2, bw);
  // with block_finish a clearly degenerate R11 is committed (the block stays
  // committed in the reference, randomized.py:253-258) and block_finish
  // raises the resample
  panel_fast(h_, mm, bw, o.Rdst, p_.ldw, o, tol_, st_, s_, true, i0, qp, true, &Mrm, &ldm, S_, ell_,
             msu, a12, 0, 0, fin_ready_ && h_.degen_commit);
  msu_ready_ = true;
  const double* Pb = p_.work + i0 + bw + i0 * p_.ldw;
  const double* Cb = p_.work + i0 + bw + (i0 + bw) * p_.ldw;
  if (!inner_gemm(h_, bw, nt2, mm - bw, Pb, p_.ldw, Cb, p_.ldw, H, bw, s2, st_, h_.num_sms - qp,
                  kProfInner))
    gemm(h_, true, false, bw, nt2, mm - bw, 1.0, Pb, p_.ldw, Cb, p_.ldw, 0.0, H, bw, s2, st_,
         kProfInner);
  RQ_CUDA(cudaEventRecord(h_.ev_join, s2));
  RQ_CUDA(cudaStreamWaitEvent(s_, h_.ev_join, 0));
  if (fin_ready_) return true;   // stages() runs block_finish()
  // G = Y_top^T C_top + M^T H   (M^T is Mrm read column-major with ld ldm)
  gemm(h_, true, false, bw, nt2, bw, 1.0, o.Y, p_.ldy, p_.work + i0 + (i0 + bw) * p_.ldw, p_.ldw,
       0.0, G_, bw, s_, st_, kProfInner);
  gemm(h_, false, false, bw, nt2, bw, 1.0, Mrm, ldm, H, bw, 1.0, G_, bw, s_, st_, kProfInner);
  fill2d(p_.work + i0 + bw + i0 * p_.ldw, p_.ldw, mm - bw, bw, 0.0, s_, st_);
  return true;
}

// `pred` is the Status predicate: a snapshot of the abort word taken before
// the block's sample update, so a degenerate verdict (which keeps this block
// committed, randomized.py:253-258) cannot skip the rows it still owes.
void Factor::trailing(int64_t i0, int64_t bw, int max_ctas, const Status* pred, cudaStream_t s) {
  const int64_t mm = m_ - i0, nt2 = n_ - i0 - bw;
  if (nt2 <= 0 || mm <= bw) return;
  if (s == nullptr) s = s_;
  const double* Yb = p_.Y + i0 + bw + i0 * p_.ldy;
  double* C = p_.work + i0 + bw + (i0 + bw) * p_.ldw;
  if (!rank_update(h_, mm - bw, nt2, bw, Yb, p_.ldy, X_, bw, C, p_.ldw, s, pred, kProfUpdate,
                   max_ctas))
    gemm(h_, false, false, mm - bw, nt2, bw, -1.0, Yb, p_.ldy, X_, bw, 1.0, C, p_.ldw, s, pred,
         kProfUpdate);
}

// SMs for the next block's select while the trailing update of the block at
// i0 runs on the rest.  The select is latency bound (64 steps of a few us,
// nearly flat in its CTA count down to ~1/3 of the GPU), the update is not:
// a ~30% share (44 of 148 SMs) measured best on cfg2 (38: 90.4 ms, 44: 88.9,
// 48: 89.1, 56: 90.4, 64: 91.9), raised where needed so every CTA's columns
// stay register-resident (<= 3 per 8-lane group of the v5 kernel, ell <= 72);
// the cluster variant (narrow samples) uses 16.
// Once the sample is narrow enough (nt <= 4608 at cfg2's b = 64, the trailing
// update then takes < 100 us), fewer columns per CTA shorten the select's
// apply phase, and 80 SMs are worth taking from the small update
// (tools/split_sweep.py: blocks 56-95 of cfg2 ~245 vs ~285 us per select phase).
int Factor::overlap_split(int64_t i0, int64_t bw) const {
  const int64_t nt1 = n_ - i0 - bw;
  const int sms = h_.num_sms;
  if (nt1 <= h_.select_cluster_max_cols) return 16;   // cluster variant
  int P = h_.overlap_sel_ctas > 0 ? h_.overlap_sel_ctas : (int)(0.30 * sms + 0.5);
  if (h_.overlap_sel_ctas <= 0) {
    // v5 (register-resident) needs <= 3 columns per 8-lane group (<= 1 for
    // ell > 72); take the SMs for it only while that stays within 80, else
    // the shared-memory v4 runs on the default share
    // v5 columns per CTA: 3 per group while the update is the longer of the
    // two, 2 (shorter apply phase, more SMs) once the select is
    int64_t per = ell_ <= 72 ? 3 * 64 : 64;
    if (ell_ <= 72 && nt1 <= h_.sel_cpg2_cols) per = 2 * 64;
    const int cap = (sms * 80) / 148;
    const int64_t need = (nt1 + per - 1) / per;
    if (need <= cap) {
      P = std::max<int64_t>(P, need);
    } else {
      // shared-memory v4: its step time grows with the columns per CTA
      // (~ell*nt1/P), the update's with its rows (~mm*nt1/(sms-P)); balance
      // the two per block.  Constant fitted on cfg5 (32768^2, ell = 136):
      // round 1, fixed 16/24/32/44/60 CTAs gave select 2366/1689/1307/949/680
      // ms and update 1072/1140/1216/1356/1591 ms per factorization; after
      // the register-held v rows (round 2) sel_balance 145/200/260/340 gave
      // 2217/2142/2163/2301 ms, and after the TMA trailing update 150/175/
      // 200/230 gave 2020/1988/1968/1958 ms (profiles/r02_cfg5_sel_balance.jsonl);
      // after the status-stream and panel changes 110/130/150/170/185/200/230/
      // 260 gave 1980/1937/1902/1882/1873/1869/1908/1989 ms (r02c_cfg5_sel_balance)
      const double mm = (double)(m_ - i0 - bw);
      P = (int)(sms / (1.0 + 1e-6 * h_.sel_balance * mm * 136.0 / (double)ell_) + 0.5);
    }
    if (nt1 <= 72 * 64) P = std::max(P, cap);
  }
  return std::max(16, std::min(P, sms - 16));
}

// Whether the next block's select outlasts this block's trailing update
// (cfg2 trace: they cross where the update is ~5 GFLOP, block ~24 of 128)
bool Factor::select_is_longer(int64_t i0, int64_t bw) const {
  const double w = 2.0 * (double)(m_ - i0 - bw) * (double)(n_ - i0 - bw) * (double)bw;
  return w < 1e-3 * (double)h_.select_main_mflop * 1e9;
}

// SMs for the fast panel while the inner product's P_below^T C_below term
// runs on the rest: fewer while that term is the longer of the two, more once
// the panel's own row chunks outnumber its CTAs (cfg2 sweep,
// tools/split_sweep.py: 32 CTAs above ~4 GFLOP of inner work, 48 down to
// ~2.6 GFLOP, then one CTA per 64-row chunk up to 80)
int Factor::panel_split(int64_t mm, int64_t nt2, int64_t bw) const {
  if (h_.overlap_panel_ctas > 0) return h_.overlap_panel_ctas;
  const double w = 2.0 * (double)(mm - bw) * (double)nt2 * (double)bw;
  const int sms = h_.num_sms;
  int q;
  if (w > 4.0e9) q = 32;
  else if (w > 2.6e9) q = 48;
  else q = (int)std::min<int64_t>((mm + 63) / 64, 80);
  q = (int)((int64_t)q * sms / 148);
  return std::max(16, std::min(q, sms - 16));
}

// D2H of the committed columns [host_done_, upto) of Y and R into the caller's
// pinned buffers on the copy stream (ordered after everything enqueued on the
// compute stream so far); `final` also takes R's columns past k.
void Factor::stream_out(int64_t upto, bool final) {
  if (p_.host_Y == nullptr && p_.host_R == nullptr) return;
  const int64_t c1 = final ? n_ : std::min(upto, n_);
  if (c1 <= host_done_) return;
  cudaStream_t cs = h_.copy_stream();
  RQ_CUDA(cudaEventRecord(h_.ev_copy, s_));
  RQ_CUDA(cudaStreamWaitEvent(cs, h_.ev_copy, 0));
  const int64_t c0 = host_done_, y1 = std::min(c1, k_);
  if (p_.host_Y != nullptr && y1 > c0)
    RQ_CUDA(cudaMemcpy2DAsync(p_.host_Y + c0 * p_.ldhY, p_.ldhY * 8, p_.Y + c0 * p_.ldy,
                              p_.ldy * 8, m_ * 8, y1 - c0, cudaMemcpyDeviceToHost, cs));
  if (p_.host_R != nullptr) {
    const double* R = p_.truncated ? p_.R : p_.work;
    const int64_t ldr = p_.truncated ? p_.ldR : p_.ldw;
    RQ_CUDA(cudaMemcpy2DAsync(p_.host_R + c0 * p_.ldhR, p_.ldhR * 8, R + c0 * ldr, ldr * 8,
                              k_ * 8, c1 - c0, cudaMemcpyDeviceToHost, cs));
  }
  host_done_ = c1;
}

// sample_update after a committed block ending at i0_new (randomized.py:253-255)
void Factor::update(int64_t i0_new, int64_t bw, bool spec, Counters& c) {
  const int64_t i0 = i0_new - bw, n2 = n_ - i0_new;
  const double *R11, *R12;
  int64_t ldr;
  if (!p_.truncated) {
    R11 = p_.work + i0 + i0 * p_.ldw; R12 = p_.work + i0 + i0_new * p_.ldw; ldr = p_.ldw;
  } else {
    R11 = p_.R + i0 + i0 * p_.ldR; R12 = p_.R + i0 + i0_new * p_.ldR; ldr = p_.ldR;
  }
  if (fin_ready_ && spec) {
    // done by block_finish()
  } else if (msu_ready_ && spec) {
    sample_update_pre(h_, ell_, bw, n2, S_, ell_, (const double*)h_.buf("su_Mpre", 8, s_), R12,
                      ldr, B_, ell_, st_, s_);
  } else {
    sample_update(h_, ell_, bw, n2, S_, ell_, R11, R12, ldr, frob_, B_, ell_, st_, spec, i0, s_);
  }
  msu_ready_ = false;
  fin_ready_ = false;
  c.gemm_flops += 3 * bw * bw * n2;
  touch(c, 2 * bw * bw + 3 * bw * n2);
}

// One block of the reference loop with host-visible branch decisions
// (randomized.py:208-258).  Returns false when the factorization stops.
// resume_panel: the speculative pass already selected and swapped this block
// (got == want) and only its fast panel declined; continue at the panel with
// the column-by-column kernel.
bool Factor::slow_block(int64_t& i0, bool resampled, int64_t& rank, bool resume_panel) {
  const int64_t want = std::min(b_, k_ - i0);
  int64_t bw = 0;
  while (true) {
    int64_t got = want;
    if (!resume_panel) {
      select(i0, want, false);
      got = read_status().got;
      if (got < want && !resampled) {
        fresh_sample(i0);
        c_.resamples += 1;
        resampled = true;
        continue;
      }
      if (got == 0) { bw = 0; break; }
      swaps(i0, got);
    }
    Counters pc;
    panel(i0, got, resampled ? kPanelCommitUsable : kPanelCommitIfFull, false, pc,
          !resume_panel && !near_floor_);
    resume_panel = false;
    c_.gemm_flops += pc.gemm_flops;
    c_.bytes_touched += pc.bytes_touched;
    const int64_t usable = read_status().usable;
    if (usable < got) near_floor_ = floor_seen_ = true;
    if (usable < got && !resampled) {
      fresh_sample(i0);
      c_.resamples += 1;
      resampled = true;
      continue;
    }
    bw = usable;
    break;
  }
  if (bw == 0) { rank = i0; return false; }
  stages(i0, bw, c_);
  i0 += bw;
  if (bw < want) { rank = i0; return false; }
  if (i0 < k_) {
    if (p_.resketch_each_block) {
      fresh_sample(i0);
    } else {
      Counters uc;
      update(i0, bw, false, uc);
      if (read_status().degenerate) {
        floor_seen_ = true;
        if (!h_.degen_commit) near_floor_ = true;
        fresh_sample(i0);
        c_.resamples += 1;
      } else {
        c_.gemm_flops += uc.gemm_flops;
        c_.bytes_touched += uc.bytes_touched;
      }
    }
  }
  return true;
}

FactorResult Factor::run() {
  m_ = p_.m; n_ = p_.n; k_ = p_.k; b_ = p_.block; ell_ = p_.ell;
  om_raw_ = p_.omega_raw;
  if (k_ < 1 || k_ > std::min(m_, n_)) throw InvalidArg("rank outside [1, min(m, n)]");
  if (ell_ > m_) throw InvalidArg("sample rows exceed matrix rows");
  if (b_ < 1 || b_ > 256) throw InvalidArg("block must be in [1, 256]");
  st_ = (Status*)h_.buf("st", sizeof(Status), s_);
  fin_done_ = (unsigned int*)h_.buf("fin_done", 64, s_);
  RQ_CUDA(cudaMemsetAsync(fin_done_, 0, 64, s_));
  pre_ = (Status*)h_.buf("st_pre", sizeof(Status), s_);
  hst_ = (Status*)h_.host_pinned("hst", sizeof(Status), s_);
  hring_ = (int*)h_.host_pinned("hring", 64 * sizeof(int), s_);
  B_ = (double*)h_.buf("sampleB", (size_t)ell_ * n_ * 8, s_);
  S_ = (double*)h_.buf("sampleS", (size_t)ell_ * n_ * 8, s_);
  piv_ = (int64_t*)h_.buf("piv", (size_t)std::max<int64_t>(b_, 1) * 8, s_);
  T_ = (double*)h_.buf("T", (size_t)b_ * b_ * 8, s_);
  G_ = (double*)h_.buf("G", (size_t)b_ * n_ * 8, s_);
  X_ = (double*)h_.buf("X", (size_t)b_ * n_ * 8, s_);
  om_d_ = (double*)h_.buf("omega_d", (size_t)ell_ * m_ * 8, s_);
  om_h_ = (double*)h_.host_pinned("omega_h", (size_t)ell_ * m_ * 8, s_);
  if (p_.truncated) {
    P_ = (double*)h_.buf("tr_panel", (size_t)m_ * b_ * 8, s_);
    Z_ = (double*)h_.buf("tr_z", (size_t)std::max(ell_, b_) * k_ * 8, s_);
  }
  RQ_CUDA(cudaMemsetAsync(st_, 0, sizeof(Status), s_));
  RQ_CUDA(cudaMemsetAsync(p_.tau, 0, (size_t)k_ * 8, s_));
  fill2d(p_.Y, p_.ldy, m_, k_, 0.0, s_);
  if (p_.truncated) {
    fill2d(p_.W, p_.ldW, n_, k_, 0.0, s_);
    fill2d(p_.R, p_.ldR, k_, n_, 0.0, s_);
  }
  {
    std::vector<int64_t> iota(n_);
    for (int64_t i = 0; i < n_; ++i) iota[i] = i;
    RQ_CUDA(cudaMemcpyAsync(p_.perm, iota.data(), n_ * 8, cudaMemcpyHostToDevice, s_));
    double* dfrob = (double*)h_.buf("frob", 8, s_);
    frob_norm(h_, p_.work, m_, n_, p_.ldw, dfrob, s_);
    RQ_CUDA(cudaMemcpyAsync(&hst_->level2, dfrob, 8, cudaMemcpyDeviceToHost, s_));
    sync();  // also keeps `iota` alive until the copy is done
    std::memcpy(&frob_, &hst_->level2, 8);
  }
  tol_ = kEps * frob_;
  fast_aborts_ = h_.fast_panel_spec != 2;
  first_sample();
  start_ahead(false);

  const bool speculate = p_.speculate && !p_.resketch_each_block;
  if (ev_.empty()) {
    ev_.resize(kLookahead + 1);
    for (auto& e : ev_) RQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  std::deque<Pending> pend;
  int slot = 0;
  const bool overlap = speculate && h_.overlap_select && !p_.truncated && p_.update_trailing;
  bool next_selected = false;   // the next block's select was launched with the previous block
  int64_t i0 = 0, rank = k_;
  bool stopped = false;
  while (true) {
    stream_out(pend.empty() ? i0 : pend.front().i0, false);   // committed columns
    // near the noise floor triggers fire block after block: queue one block
    // ahead only, so a rewind discards fewer (early-exiting) launches
    const int ahead =
        floor_seen_ ? std::max(1, std::min(kLookahead, h_.floor_lookahead)) : kLookahead;
    if (!pend.empty() && (stopped || i0 >= k_ || (int)pend.size() >= ahead)) {
      Pending e = pend.front();
      RQ_CUDA(cudaEventSynchronize(ev_[e.slot]));
      if (hring_[e.slot] != 0) {
        // a trigger fired at or after block e.i0: rewind to it
        const Status stt = read_status();
        const int64_t X = stt.abort_i0;
        const int code = stt.abort;
        int64_t bwX = 0;
        for (const Pending& q : pend) {
          if (q.i0 < X) {
            c_.gemm_flops += q.stage.gemm_flops + q.update.gemm_flops;
            c_.bytes_touched += q.stage.bytes_touched + q.update.bytes_touched;
          } else if (q.i0 == X) {
            bwX = q.bw;
            if (code == kAbortDegenerate) {
              c_.gemm_flops += q.stage.gemm_flops;
              c_.bytes_touched += q.stage.bytes_touched;
            }
          }
        }
        pend.clear();
        if (overlap) RQ_CUDA(cudaStreamSynchronize(h_.side_stream()));
        next_selected = false;
        msu_ready_ = fin_ready_ = false;
        RQ_CUDA(cudaMemsetAsync(&st_->abort, 0, sizeof(int), s_));
        if (code == kAbortDegenerate || code == kAbortPanelFast || code == kAbortPanelRank)
          floor_seen_ = true;
        // a degenerate verdict no longer dooms the fast panel (it commits a
        // clearly degenerate R11); a declined fast panel or a rank cut does
        if (code == kAbortPanelFast || code == kAbortPanelRank ||
            (code == kAbortDegenerate && !h_.degen_commit))
          near_floor_ = true;
        if (code == kAbortDegenerate) {
          i0 = X + bwX;
          fresh_sample(i0);
          c_.resamples += 1;
        } else if (code == kAbortPanelFast) {
          // not a reference branch: block X's select and swaps stand, only
          // its panel is redone column by column
          i0 = X;
          fast_aborts_ = h_.fast_panel_spec == 0;
          if (!slow_block(i0, false, rank, true)) { stopped = true; break; }
        } else {
          i0 = X;
          fresh_sample(i0);
          c_.resamples += 1;
          if (!slow_block(i0, true, rank)) { stopped = true; break; }
        }
        continue;
      }
      c_.gemm_flops += e.stage.gemm_flops + e.update.gemm_flops;
      c_.bytes_touched += e.stage.bytes_touched + e.update.bytes_touched;
      pend.pop_front();
      continue;
    }
    if (stopped || i0 >= k_) break;
    if (!speculate) {
      if (!slow_block(i0, false, rank)) { stopped = true; }
      continue;
    }
    // ---- speculative block: assume got == usable == want, no degenerate R11
    const int64_t want = std::min(b_, k_ - i0);
    Pending e{};
    e.i0 = i0;
    e.bw = want;
    if (!next_selected) select(i0, want, true);   // else launched during the previous block
    next_selected = false;
    swaps(i0, want);
    msu_ready_ = fin_ready_ = false;
    const bool g_ready = overlap && h_.overlap_inner && fast_aborts_ && !near_floor_ &&
                         panel_overlap_inner(i0, want);
    if (!g_ready) panel(i0, want, kPanelCommitIfFull, true, e.stage, !near_floor_);
    e.has_update = i0 + want < k_;
    // RQRCP: the next block's select only needs the sample update (R11, R12),
    // so it runs on a side stream on a share of the SMs while the trailing
    // rows of this block's update run on the rest (join before its swaps)
    const bool ovl = overlap && e.has_update && m_ - i0 > want;
    stages(i0, want, e.stage, ovl, g_ready);   // with ovl, also snapshots the abort word
    if (e.has_update) update(i0 + want, want, true, e.update);
    if (ovl) {
      const int P = overlap_split(i0, want);
      cudaStream_t s2 = h_.side_stream();
      RQ_CUDA(cudaEventRecord(h_.ev_fork, s_));
      RQ_CUDA(cudaStreamWaitEvent(s2, h_.ev_fork, 0));
      // the longer of the two stays on the main stream, so the chain
      // select -> swaps -> panel (or update -> swaps) has no cross-stream hop
      if (h_.select_on_main && select_is_longer(i0, want)) {
        trailing(i0, want, h_.num_sms - P, pre_, s2);
        select(i0 + want, std::min(b_, k_ - i0 - want), true, s_, P);
      } else {
        select(i0 + want, std::min(b_, k_ - i0 - want), true, s2, P);
        trailing(i0, want, h_.num_sms - P, pre_);
      }
      RQ_CUDA(cudaEventRecord(h_.ev_join, s2));
      RQ_CUDA(cudaStreamWaitEvent(s_, h_.ev_join, 0));
      next_selected = true;
    }
    e.slot = slot;
    // abort-word snapshot for the host's retire check, off the compute stream
    // (it may also see a later block's trigger: the rewind below takes the
    // block from Status, not from the slot)
    {
      cudaStream_t ss = h_.stat_stream();
      RQ_CUDA(cudaEventRecord(h_.ev_stat, s_));
      RQ_CUDA(cudaStreamWaitEvent(ss, h_.ev_stat, 0));
      RQ_CUDA(cudaMemcpyAsync(&hring_[slot], &st_->abort, sizeof(int), cudaMemcpyDeviceToHost, ss));
      RQ_CUDA(cudaEventRecord(ev_[slot], ss));
    }
    slot = (slot + 1) % (kLookahead + 1);
    pend.push_back(e);
    i0 += want;
  }
  const Status fin = read_status();
  if (speculate) RQ_CUDA(cudaStreamSynchronize(h_.stat_stream()));
  stream_out(n_, true);
  if (p_.host_Y != nullptr || p_.host_R != nullptr)
    RQ_CUDA(cudaStreamSynchronize(h_.copy_stream()));
  FactorResult r;
  r.rank = rank;
  r.nswaps = fin.nswaps;
  r.c = c_;
  r.c.level2_flops = fin.level2;
  r.c.bytes_touched += fin.l2bytes;
  r.frob = frob_;
  return r;
}

}  // namespace

FactorResult run_factor(Handle& h, const FactorParams& p) {
  Factor f(h, p);
  return f.run();
}

// ------------------------------------------------------------------ qr_blocked / q_columns

void qr_blocked(Handle& h, int64_t m, int64_t n, int64_t k, int64_t b, double* work,
                int64_t ldw, double* Y, int64_t ldy, double* tau, Counters* c, cudaStream_t s) {
  if (b < 1 || b > 256) throw InvalidArg("block must be in [1, 256]");
  Status* st = (Status*)h.buf("qr_st", sizeof(Status), s);
  RQ_CUDA(cudaMemsetAsync(st, 0, sizeof(Status), s));
  fill2d(Y, ldy, m, k, 0.0, s);
  RQ_CUDA(cudaMemsetAsync(tau, 0, (size_t)std::max<int64_t>(k, 1) * 8, s));
  double* T = (double*)h.buf("qr_T", (size_t)b * b * 8, s);
  double* G = (double*)h.buf("qr_G", (size_t)b * std::max<int64_t>(n, 1) * 8, s);
  double* X = (double*)h.buf("qr_X", (size_t)b * std::max<int64_t>(n, 1) * 8, s);
  for (int64_t i0 = 0; i0 < k; i0 += b) {
    const int64_t bw = std::min(b, k - i0), mm = m - i0, nc = n - i0 - bw;
    PanelOut o{};
    o.Rdst = work + i0 + i0 * ldw; o.ldr = ldw; o.rrows = mm;
    o.Y = Y + i0 + i0 * ldy; o.ldy = ldy; o.tau = tau + i0;
    o.T = nc > 0 ? T : nullptr; o.ldt = b;
    panel_qr(h, mm, bw, work + i0 + i0 * ldw, ldw, o, -1.0, kPanelCommitAll, false, st, i0, s);
    if (nc > 0) {
      // apply_block_reflection(transpose=True) (kernels.py:166-181)
      double* C = work + i0 + (i0 + bw) * ldw;
      const double* Yb = Y + i0 + i0 * ldy;
      if (!inner_gemm(h, bw, nc, mm, Yb, ldy, C, ldw, G, bw, s, nullptr, 0, kProfInner))
        gemm(h, true, false, bw, nc, mm, 1.0, Yb, ldy, C, ldw, 0.0, G, bw, s);
      gemm(h, true, false, bw, nc, bw, 1.0, T, b, G, bw, 0.0, X, bw, s);
      gemm(h, false, false, mm, nc, bw, -1.0, Yb, ldy, X, bw, 1.0, C, ldw, s);
      if (c) {
        c->gemm_flops += 4 * mm * bw * nc + bw * bw * nc;
        c->bytes_touched += 8 * (2 * mm * nc + mm * bw + bw * nc);
      }
    }
  }
  if (c) {
    Status hs;
    RQ_CUDA(cudaMemcpyAsync(&hs, st, sizeof(Status), cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    c->level2_flops += hs.level2;
    c->bytes_touched += hs.l2bytes;
  }
}

void q_columns(Handle& h, int64_t m, int64_t nref, int64_t cols, const double* Y, int64_t ldy,
               const double* tau, int64_t b, double* Q, int64_t ldq, cudaStream_t s) {
  set_identity(Q, ldq, m, cols, s);
  if (nref <= 0 || cols <= 0) return;
  double* T = (double*)h.buf("qc_T", (size_t)b * b * 8, s);
  double* G = (double*)h.buf("qc_G", (size_t)b * cols * 8, s);
  double* X = (double*)h.buf("qc_X", (size_t)b * cols * 8, s);
  const int64_t nblk = (nref + b - 1) / b;
  for (int64_t J = nblk - 1; J >= 0; --J) {
    const int64_t i0 = J * b, bw = std::min(b, nref - i0), mm = m - i0;
    if (i0 >= cols) continue;  // columns < i0 are untouched identity columns
    const int64_t nc = cols - i0;
    const double* Yb = Y + i0 + i0 * ldy;
    t_factor(h, Yb, ldy, mm, bw, tau + i0, T, b, s);
    double* C = Q + i0 + i0 * ldq;
    if (!inner_gemm(h, bw, nc, mm, Yb, ldy, C, ldq, G, bw, s, nullptr, 0, kProfInner))
      gemm(h, true, false, bw, nc, mm, 1.0, Yb, ldy, C, ldq, 0.0, G, bw, s);
    gemm(h, false, false, bw, nc, bw, 1.0, T, b, G, bw, 0.0, X, bw, s);
    gemm(h, false, false, mm, nc, bw, -1.0, Yb, ldy, X, bw, 1.0, C, ldq, s);
  }
}

}  // namespace rq

namespace rq {

// ------------------------------------------------------------------ TUXV
TuxvResult run_tuxv(Handle& h, const TuxvParams& p) {
  if (p.j_max < 1) throw InvalidArg("j_max must be >= 1");
  cudaStream_t s = p.f.stream;
  TuxvResult out;
  out.f = run_factor(h, p.f);
  Counters c = out.f.c;
  const int64_t m = p.f.m, n = p.f.n, r = out.f.rank, b = p.f.block;
  out.rank = r;
  if (r == 0) {
    out.f.c = c;
    return out;
  }
  // Z = perm.restore(R[:r]) (k x n -> r x n), then lq_factor(Z) = qr_blocked(Z^T)
  double* Z = (double*)h.buf("tx_Z", (size_t)r * n * 8, s);
  fill2d(Z, r, r, n, 0.0, s);
  scatter_cols(p.f.R, p.f.ldR, p.f.perm, Z, r, r, n, s);
  double* Zt = (double*)h.buf("tx_Zt", (size_t)std::max(m, n) * r * 8, s);
  double* Yq = (double*)h.buf("tx_Yq", (size_t)std::max(m, n) * r * 8, s);
  double* tq = (double*)h.buf("tx_tau", (size_t)r * 8, s);
  transpose(Z, r, Zt, n, r, n, s);
  qr_blocked(h, n, r, r, b, Zt, n, Yq, n, tq, &c, s);
  q_columns(h, n, r, r, Yq, n, tq, b, p.V, p.ldv, s);
  int64_t j = 1;
  while (true) {
    // Zc = A V[:, :r]; U, X from qr_blocked(Zc)
    gemm(h, false, false, m, r, n, 1.0, p.A, p.lda, p.V, p.ldv, 0.0, Zt, m, s);
    c.gemm_flops += 2 * m * n * r;
    c.bytes_touched += 8 * (m * n + n * r + m * r);
    qr_blocked(h, m, r, r, b, Zt, m, Yq, m, tq, &c, s);
    q_columns(h, m, r, r, Yq, m, tq, b, p.U, p.ldu, s);
    copy2d(Zt, m, p.X, p.ldx, r, r, s);
    out.x_lower = 0;
    if (j >= p.j_max) break;
    // Zr = U^T A (r x n); X, V = lq_factor(Zr)
    gemm(h, true, false, r, n, m, 1.0, p.U, p.ldu, p.A, p.lda, 0.0, Z, r, s);
    c.gemm_flops += 2 * m * n * r;
    c.bytes_touched += 8 * (m * r + r * n);
    transpose(Z, r, Zt, n, r, n, s);
    qr_blocked(h, n, r, r, b, Zt, n, Yq, n, tq, &c, s);
    q_columns(h, n, r, r, Yq, n, tq, b, p.V, p.ldv, s);
    transpose(Zt, n, p.X, p.ldx, r, r, s);  // L = R^T
    out.x_lower = 1;
    if (j + 1 >= p.j_max) break;
    j += 2;
  }
  RQ_CUDA(cudaStreamSynchronize(s));
  out.f.c = c;
  return out;
}

}  // namespace rq
