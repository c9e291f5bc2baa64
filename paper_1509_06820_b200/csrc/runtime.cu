// Host runtime: handle, workspace arena, launch counter and the optional
// CUDA-event profiler used by bench.py.
#include <atomic>
#include <mutex>
#include <tuple>

#include "runtime.hpp"

namespace rq {

namespace {
std::atomic<int64_t> g_launches{0};
std::mutex g_attr_mu;
std::map<std::tuple<const void*, int, int>, int> g_attrs;
}

void kernel_attr(const void* func, cudaFuncAttribute attr, int value) {
  int dev = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_attr_mu);
  const auto key = std::make_tuple(func, dev, (int)attr);
  auto it = g_attrs.find(key);
  if (it != g_attrs.end() &&
      (attr == cudaFuncAttributeMaxDynamicSharedMemorySize ? it->second >= value
                                                            : it->second == value))
    return;
  RQ_CUDA(cudaFuncSetAttribute(func, attr, value));
  g_attrs[key] = value;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

ProfScope::ProfScope(Handle& h, int cat, double flops, double bytes, cudaStream_t s)
    : h_(&h), s_(s) {
  if (h.profiling && cat >= 0) idx_ = h.prof_begin(cat, flops, bytes, s);   // cat < 0: untimed
}
ProfScope::~ProfScope() {
  if (idx_ >= 0) h_->prof_end(idx_, s_);
}

cudaEvent_t Handle::take_event() {
  if (free_ev_.empty()) {
    cudaEvent_t e;
    RQ_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = free_ev_.back();
  free_ev_.pop_back();
  return e;
}

int Handle::prof_begin(int cat, double flops, double bytes, cudaStream_t s) {
  PendEv p{cat, flops, bytes, take_event(), take_event()};
  RQ_CUDA(cudaEventRecord(p.a, s));
  pend_.push_back(p);
  return (int)pend_.size() - 1;
}

void Handle::prof_end(int idx, cudaStream_t s) { RQ_CUDA(cudaEventRecord(pend_[idx].b, s)); }

void Handle::prof_collect() {
  for (auto& p : pend_) {
    RQ_CUDA(cudaEventSynchronize(p.b));
    float ms = 0.f;
    RQ_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    if (tracing && trace_base_ != nullptr) {
      float t0 = 0.f;
      RQ_CUDA(cudaEventElapsedTime(&t0, trace_base_, p.a));
      trace.push_back({p.cat, (double)t0, (double)t0 + ms});
    }
    ProfStat& st = stats[p.cat];
    st.launches += 1;
    st.ms += ms;
    st.flops += p.flops;
    st.bytes += p.bytes;
    free_ev_.push_back(p.a);
    free_ev_.push_back(p.b);
  }
  pend_.clear();
}

void Handle::prof_reset() {
  prof_collect();
  for (auto& s : stats) s = ProfStat{};
  trace.clear();
  if (tracing) {
    if (trace_base_ == nullptr) RQ_CUDA(cudaEventCreate(&trace_base_));
    RQ_CUDA(cudaEventRecord(trace_base_, 0));
  }
}

// ------------------------------------------------------------------ Handle
Handle::Handle(int dev) : device(dev) {
  RQ_CUDA(cudaSetDevice(dev));
  RQ_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  int optin = 0;
  RQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  smem_optin = (size_t)optin;
}

cudaStream_t Handle::side_stream() {
  if (side_ == nullptr) {
    RQ_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    RQ_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    RQ_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  }
  return side_;
}

cudaStream_t Handle::copy_stream() {
  if (copy_ == nullptr) {
    RQ_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
    RQ_CUDA(cudaEventCreateWithFlags(&ev_copy, cudaEventDisableTiming));
  }
  return copy_;
}

cudaStream_t Handle::stat_stream() {
  if (stat_ == nullptr) {
    RQ_CUDA(cudaStreamCreateWithFlags(&stat_, cudaStreamNonBlocking));
    RQ_CUDA(cudaEventCreateWithFlags(&ev_stat, cudaEventDisableTiming));
  }
  return stat_;
}

cudaStream_t Handle::omega_stream() {
  if (omega_ == nullptr) {
    RQ_CUDA(cudaStreamCreateWithFlags(&omega_, cudaStreamNonBlocking));
    RQ_CUDA(cudaEventCreateWithFlags(&ev_omega, cudaEventDisableTiming));
  }
  return omega_;
}

Handle::~Handle() {
  if (omega_ != nullptr) {
    cudaStreamDestroy(omega_);
    cudaEventDestroy(ev_omega);
  }
  if (stat_ != nullptr) {
    cudaStreamDestroy(stat_);
    cudaEventDestroy(ev_stat);
  }
  if (copy_ != nullptr) {
    cudaStreamDestroy(copy_);
    cudaEventDestroy(ev_copy);
  }
  if (side_ != nullptr) {
    cudaStreamDestroy(side_);
    cudaEventDestroy(ev_fork);
    cudaEventDestroy(ev_join);
  }
  for (auto e : ring_ev) cudaEventDestroy(e);
  for (auto e : free_ev_) cudaEventDestroy(e);
  for (auto& p : pend_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto& kv : bufs_) {
    if (!kv.second.p) continue;
    if (kv.second.pinned) cudaFreeHost(kv.second.p);
    else cudaFree(kv.second.p);
  }
}

void* Handle::buf(const std::string& name, size_t bytes, cudaStream_t s) {
  Buf& b = bufs_[name];
  if (bytes == 0) bytes = 8;
  if (b.bytes < bytes) {
    if (b.p) {
      RQ_CUDA(cudaStreamSynchronize(s));
      RQ_CUDA(cudaFree(b.p));
      b.p = nullptr;
    }
    RQ_CUDA(cudaMalloc(&b.p, bytes));
    b.bytes = bytes;
  }
  return b.p;
}

void* Handle::host_pinned(const std::string& name, size_t bytes, cudaStream_t s) {
  Buf& b = bufs_["host:" + name];
  if (bytes == 0) bytes = 8;
  if (b.bytes < bytes) {
    if (b.p) {
      RQ_CUDA(cudaStreamSynchronize(s));
      RQ_CUDA(cudaFreeHost(b.p));
      b.p = nullptr;
    }
    RQ_CUDA(cudaMallocHost(&b.p, bytes));
    b.bytes = bytes;
    b.pinned = true;
  }
  return b.p;
}

}  // namespace rq
