// extern "C" boundary (include/rqrcp_b200.h): argument checks, exception ->
// status-code mapping, and the thin adapters onto the native drivers.
#include <mutex>
#include <string>

#include "../../include/rqrcp_b200.h"
#include "driver.hpp"

struct rq_handle_s {
  rq::Handle* h;
  std::recursive_mutex mu;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    g_err.clear();
    f();
    return RQ_OK;
  } catch (const rq::InvalidArg& e) {
    g_err = e.what();
    return RQ_ERR_INVALID;
  } catch (const rq::CudaError& e) {
    g_err = e.what();
    return RQ_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RQ_ERR_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return RQ_ERR_INTERNAL;
  }
}

// Every call on a handle runs with the handle's device current and puts the
// caller's current device back afterwards (a process may drive several GPUs,
// one handle each; PyTorch keeps its own notion of the current device).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) RQ_CUDA(cudaSetDevice(dev));
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// calls on one handle are serialised: its named scratch buffers and Status
// word are shared by every call on that device
template <class F>
int guarded_on(rq_handle_t h, F&& f) {
  return guarded([&] {
    if (h == nullptr || h->h == nullptr) throw rq::InvalidArg("null handle");
    std::lock_guard<std::recursive_mutex> lock(h->mu);
    DeviceScope dev(h->h->device);
    f();
  });
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void need(bool ok, const char* what) {
  if (!ok) throw rq::InvalidArg(what);
}

rq::Handle& H(rq_handle_t h) {
  need(h != nullptr && h->h != nullptr, "null handle");
  return *h->h;
}

rq::FactorParams to_params(const rq_factor_args& a) {
  need(a.m >= 1 && a.n >= 1, "matrix must be non-empty");
  need(a.k >= 1 && a.k <= std::min(a.m, a.n), "rank must be >= 1 and <= min(m, n)");
  need(a.ell >= 1 && a.ell <= a.m, "sample rows exceed matrix rows");
  need(a.block >= 1, "block must be >= 1");
  need(a.work && a.Y && a.tau && a.perm && a.swaps, "null output buffer");
  need(a.ldw >= a.m && a.ldy >= a.m, "leading dimension too small");
  rq::FactorParams p;
  p.m = a.m; p.n = a.n; p.k = a.k; p.block = a.block; p.ell = a.ell;
  p.resketch_each_block = a.variant == RQ_RSRQRCP;
  p.update_trailing = a.variant == RQ_RQRCP || a.variant == RQ_RSRQRCP;
  p.truncated = a.variant == RQ_TRQRCP;
  if (p.truncated) {
    need(a.W && a.R, "TRQRCP needs W and R buffers");
    need(a.ldW >= a.n && a.ldR >= a.k, "leading dimension too small");
  }
  p.work = a.work; p.ldw = a.ldw; p.Y = a.Y; p.ldy = a.ldy; p.tau = a.tau;
  p.W = a.W; p.ldW = a.ldW; p.R = a.R; p.ldR = a.ldR;
  p.perm = a.perm; p.swaps = a.swaps; p.swap_cap = a.swap_cap;
  p.omega0 = a.omega0; p.omega_fn = a.omega_fn; p.omega_user = a.omega_user;
  p.speculate = a.speculate;
  p.stream = S(a.stream);
  p.host_Y = a.host_Y; p.ldhY = a.ldhY;
  p.host_R = a.host_R; p.ldhR = a.ldhR;
  p.omega_native = a.omega_native != 0;
  p.omega_threads = a.omega_threads;
  p.omega_k0 = a.omega_k0; p.omega_k1 = a.omega_k1; p.omega_raw = a.omega_raw;
  return p;
}

void fill_result(const rq::FactorResult& r, rq_factor_result* out) {
  out->rank = r.rank;
  out->nswaps = r.nswaps;
  out->gemm_flops = r.c.gemm_flops;
  out->level2_flops = r.c.level2_flops;
  out->bytes_touched = r.c.bytes_touched;
  out->resamples = r.c.resamples;
  out->frob = r.frob;
}

}  // namespace

extern "C" {

int rq_version(void) { return 100; }

const char* rq_last_error(void) { return g_err.c_str(); }

int rq_create(int device, rq_handle_t* out) {
  return guarded([&] {
    need(out != nullptr, "null output");
    auto* h = new rq_handle_s;
    try {
      DeviceScope dev(device);   // the caller's current device is left as it was
      h->h = new rq::Handle(device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int rq_destroy(rq_handle_t h) {
  return guarded([&] {
    if (!h) return;
    {
      DeviceScope dev(h->h->device);
      delete h->h;
    }
    delete h;
  });
}

int rq_factor(rq_handle_t h, const rq_factor_args* args, rq_factor_result* out) {
  return guarded_on(h, [&] {
    need(args && out, "null argument");
    rq::FactorParams p = to_params(*args);
    rq::FactorResult r = rq::run_factor(H(h), p);
    fill_result(r, out);
  });
}

int rq_tuxv(rq_handle_t h, const rq_tuxv_args* args, rq_tuxv_result* out) {
  return guarded_on(h, [&] {
    need(args && out, "null argument");
    need(args->f.variant == RQ_TRQRCP, "tuxv runs on TRQRCP");
    need(args->j_max >= 1, "j_max must be >= 1");
    need(args->A && args->U && args->V && args->X, "null output buffer");
    rq::TuxvParams p;
    p.f = to_params(args->f);
    p.A = args->A; p.lda = args->lda; p.j_max = args->j_max;
    p.U = args->U; p.ldu = args->ldu; p.V = args->V; p.ldv = args->ldv;
    p.X = args->X; p.ldx = args->ldx;
    rq::TuxvResult r = rq::run_tuxv(H(h), p);
    fill_result(r.f, &out->f);
    out->rank = r.rank;
    out->x_lower = r.x_lower;
  });
}

int rq_gemm(rq_handle_t h, int transa, int transb, int64_t m, int64_t n, int64_t k,
            double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
            double beta, double* C, int64_t ldc, void* stream) {
  return guarded_on(h, [&] {
    need(m >= 0 && n >= 0 && k >= 0, "negative dimension");
    need(ldc >= std::max<int64_t>(1, m), "ldc too small");
    rq::gemm(H(h), transa != 0, transb != 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
             S(stream));
  });
}

int rq_sketch(rq_handle_t h, int64_t ell, int64_t m, int64_t n, const double* omega,
              int64_t ldo, const double* A, int64_t lda, double* B, int64_t ldb, void* stream) {
  return guarded_on(h, [&] {
    need(ell >= 1, "sample must have at least one row");
    rq::gemm(H(h), false, false, ell, n, m, 1.0, omega, ldo, A, lda, 0.0, B, ldb, S(stream));
  });
}

int rq_select_pivots(rq_handle_t h, int64_t ell, int64_t nt, int64_t want, const double* B,
                     int64_t ldb, double* S_, int64_t lds, int64_t* piv, double* Ys,
                     int64_t ldys, double* taus, int64_t* got, int64_t* level2,
                     void* stream) {
  return guarded_on(h, [&] {
    rq::Handle& hh = H(h);
    cudaStream_t s = S(stream);
    auto* st = (rq::Status*)hh.buf("abi_st", sizeof(rq::Status), s);
    RQ_CUDA(cudaMemsetAsync(st, 0, sizeof(rq::Status), s));
    rq::SelectOut o{S_, lds, piv, Ys, ldys, taus};
    rq::select_pivots(hh, ell, nt, want, B, ldb, o, st, false, 0, s);
    rq::Status hs;
    RQ_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    if (got) *got = hs.got;
    if (level2) *level2 = hs.level2;
  });
}

int rq_panel_qr(rq_handle_t h, int64_t mm, int64_t bw, double* P, int64_t ldp, double* Y,
                int64_t ldy, double* tau, double* T, int64_t ldt, double tol, int64_t* usable,
                int64_t* level2, void* stream) {
  return guarded_on(h, [&] {
    rq::Handle& hh = H(h);
    cudaStream_t s = S(stream);
    auto* st = (rq::Status*)hh.buf("abi_st", sizeof(rq::Status), s);
    RQ_CUDA(cudaMemsetAsync(st, 0, sizeof(rq::Status), s));
    rq::PanelOut o{P, ldp, mm, Y, ldy, tau, T, ldt};
    rq::panel_qr(hh, mm, bw, P, ldp, o, tol, rq::kPanelCommitAll, false, st, 0, s);
    rq::Status hs;
    RQ_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    if (usable) *usable = hs.usable;
    if (level2) *level2 = hs.level2;
  });
}

int rq_t_factor(rq_handle_t h, const double* Y, int64_t ldy, int64_t mm, int64_t nb,
                const double* tau, double* T, int64_t ldt, void* stream) {
  return guarded_on(h, [&] { rq::t_factor(H(h), Y, ldy, mm, nb, tau, T, ldt, S(stream)); });
}

int rq_sample_update(rq_handle_t h, int64_t ell, int64_t b, int64_t n2, const double* S_,
                     int64_t lds, const double* R11, const double* R12, int64_t ldr,
                     double frob, double* Bnew, int64_t ldb, int32_t* degenerate,
                     void* stream) {
  return guarded_on(h, [&] {
    rq::Handle& hh = H(h);
    cudaStream_t s = S(stream);
    auto* st = (rq::Status*)hh.buf("abi_st", sizeof(rq::Status), s);
    RQ_CUDA(cudaMemsetAsync(st, 0, sizeof(rq::Status), s));
    rq::sample_update(hh, ell, b, n2, S_, lds, R11, R12, ldr, frob, Bnew, ldb, st, false, 0, s);
    rq::Status hs;
    RQ_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    if (degenerate) *degenerate = (int32_t)hs.degenerate;
  });
}

int rq_qr_blocked(rq_handle_t h, int64_t m, int64_t n, int64_t k, int64_t b, double* A,
                  int64_t lda, double* Y, int64_t ldy, double* tau, int64_t* counters,
                  void* stream) {
  return guarded_on(h, [&] {
    need(k >= 0 && k <= std::min(m, n), "rank outside [0, min(m, n)]");
    need(b >= 1, "block size must be >= 1");
    rq::Counters c;
    rq::qr_blocked(H(h), m, n, k, b, A, lda, Y, ldy, tau, &c, S(stream));
    if (counters) {
      counters[0] += c.gemm_flops;
      counters[1] += c.level2_flops;
      counters[2] += c.bytes_touched;
    }
  });
}

int rq_q_columns(rq_handle_t h, int64_t m, int64_t nref, int64_t cols, const double* Y,
                 int64_t ldy, const double* tau, int64_t b, double* Q, int64_t ldq,
                 void* stream) {
  return guarded_on(h, [&] {
    need(b >= 1, "block size must be >= 1");
    rq::q_columns(H(h), m, nref, cols, Y, ldy, tau, b, Q, ldq, S(stream));
  });
}

int rq_column_norms(rq_handle_t h, const double* A, int64_t m, int64_t n, int64_t lda,
                    int sequential, double* out, void* stream) {
  return guarded_on(h, [&] {
    need(m >= 0 && n >= 0 && lda >= std::max<int64_t>(m, 1), "bad shape");
    rq::column_norms(H(h), A, m, n, lda, sequential != 0, out, S(stream));
  });
}

int rq_frob_norm(rq_handle_t h, const double* A, int64_t m, int64_t n, int64_t lda,
                 double* out, void* stream) {
  return guarded_on(h, [&] { rq::frob_norm(H(h), A, m, n, lda, out, S(stream)); });
}

int rq_downdate_norms(rq_handle_t h, const double* norms, const double* row, int64_t inc,
                      int64_t n, const double* orig_sq, double guard, double* out,
                      int32_t* unsafe, void* stream) {
  return guarded_on(h, [&] {
    need(n >= 0 && inc >= 1, "bad shape");
    need(norms != nullptr && row != nullptr && out != nullptr, "null argument");
    rq::downdate_norms(norms, row, inc, n, orig_sq, guard, out, unsafe, S(stream));
  });
}

int64_t rq_launch_count(void) { return rq::launch_count(); }

int rq_set_option(rq_handle_t h, const char* name, int64_t value) {
  return guarded_on(h, [&] {
    need(name != nullptr, "null option name");
    rq::Handle& hh = H(h);
    const std::string n(name);
    if (n == "force_select") hh.force_select = (int)value;
    else if (n == "force_panel") hh.force_panel = (int)value;
    else if (n == "select_cluster_max_cols") hh.select_cluster_max_cols = value;
    else if (n == "panel_cluster_max_rows") hh.panel_cluster_max_rows = value;
    else if (n == "panel_rows_per_cta") hh.panel_rows_per_cta = std::max<int64_t>(32, value);
    else if (n == "use_rank_update") hh.use_rank_update = value != 0;
    else if (n == "fast_panel") hh.fast_panel = value != 0;
    else if (n == "fast_panel_max_ctas") hh.fast_panel_max_ctas = (int)value;
    else if (n == "fast_panel_pad") hh.fast_panel_pad = (int)std::max<int64_t>(1, std::min<int64_t>(value, 8));
    else if (n == "fast_panel_spec") hh.fast_panel_spec = (int)value;
    else if (n == "profile_trace") hh.tracing = value != 0;
    else if (n == "select_max_ctas") hh.select_max_ctas = (int)value;
    else if (n == "select_reg") hh.select_reg = value != 0;
    else if (n == "select_fused") hh.select_fused = value != 0;
    else if (n == "omega_ahead") hh.omega_ahead = value != 0;
    else if (n == "floor_lookahead") hh.floor_lookahead = (int)value;
    else if (n == "t_inverse") hh.t_inverse = value != 0;
    else if (n == "panel_halves") hh.panel_halves = value != 0;
    else if (n == "degen_commit") hh.degen_commit = value != 0;
    else if (n == "finish_narrow") hh.finish_narrow = value != 0;
    else if (n == "use_tc") hh.use_tc = value != 0;
    else if (n == "tc_variant") hh.tc_variant = (int)value;
    else if (n == "tc_splits") hh.tc_splits = (int)value;
    else if (n == "tc_tma") hh.tc_tma = value != 0;
    else if (n == "overlap_select") hh.overlap_select = value != 0;
    else if (n == "overlap_sel_ctas") hh.overlap_sel_ctas = (int)value;
    else if (n == "select_on_main") hh.select_on_main = value != 0;
    else if (n == "select_main_mflop") hh.select_main_mflop = (int)value;
    else if (n == "sel_cpg2_cols") hh.sel_cpg2_cols = value;
    else if (n == "sel_balance") hh.sel_balance = (int)value;
    else if (n == "su_gemm") hh.su_gemm = value != 0;
    else if (n == "overlap_inner") hh.overlap_inner = value != 0;
    else if (n == "overlap_panel_ctas") hh.overlap_panel_ctas = (int)value;
    else if (n == "block_finish") hh.block_finish = value != 0;
    else if (n == "ru_two_ctas") hh.ru_two_ctas = value != 0;
    else if (n == "ru_skew_ns") hh.ru_skew_ns = (int)value;
    else if (n == "ru_big") hh.ru_big = value != 0;
    else if (n == "ru_tma") hh.ru_tma = (int)value;
    else if (n == "inner_kernel") hh.inner_kernel = value != 0;
    else if (n == "inner_ktiles") hh.inner_ktiles = (int)value;
    else if (n == "inner32") hh.inner32 = value != 0;
    else if (n == "gemm_vec16") hh.gemm_vec16 = value != 0;
    else if (n == "debug_timers") {
      hh.dbg = value ? (long long*)hh.buf("dbg_timers", 64 * 8, nullptr) : nullptr;
      if (hh.dbg) RQ_CUDA(cudaMemset(hh.dbg, 0, 64 * 8));
    }
    else throw rq::InvalidArg("unknown option " + n);
  });
}

int rq_debug_read(rq_handle_t h, int64_t* out, int n) {
  return guarded_on(h, [&] {
    rq::Handle& hh = H(h);
    need(hh.dbg != nullptr, "debug timers not enabled");
    RQ_CUDA(cudaDeviceSynchronize());
    RQ_CUDA(cudaMemcpy(out, hh.dbg, (size_t)std::min(n, 64) * 8, cudaMemcpyDeviceToHost));
  });
}

int rq_profile_enable(rq_handle_t h, int on) {
  return guarded_on(h, [&] { H(h).profiling = on != 0; });
}

int rq_profile_reset(rq_handle_t h) {
  return guarded_on(h, [&] { H(h).prof_reset(); });
}

int rq_profile_read(rq_handle_t h, int64_t* launches, double* ms, double* flops, double* bytes) {
  return guarded_on(h, [&] {
    rq::Handle& hh = H(h);
    hh.prof_collect();
    for (int i = 0; i < rq::kProfNum; ++i) {
      if (launches) launches[i] = hh.stats[i].launches;
      if (ms) ms[i] = hh.stats[i].ms;
      if (flops) flops[i] = hh.stats[i].flops;
      if (bytes) bytes[i] = hh.stats[i].bytes;
    }
  });
}

}  // extern "C"

int rq_profile_trace(rq_handle_t h, int64_t cap, int32_t* cat, double* start_ms, double* end_ms,
                     int64_t* count) {
  return guarded_on(h, [&] {
    rq::Handle& hh = H(h);
    hh.prof_collect();
    const int64_t nrec = (int64_t)hh.trace.size();
    for (int64_t i = 0; i < nrec && i < cap; ++i) {
      cat[i] = hh.trace[i].cat;
      start_ms[i] = hh.trace[i].start_ms;
      end_ms[i] = hh.trace[i].end_ms;
    }
    *count = nrec;
  });
}
