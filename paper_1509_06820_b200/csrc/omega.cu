// Host Omega stream (rng.py:16-41 of the reference: RngState(seed) wraps
// numpy's Philox(key=seed) and draws standard_normal; Omega is that stream
// filled column-major).  Omega stays host-generated, as the north star asks;
// this file only makes the draw multi-threaded while keeping every value
// bit-identical to numpy's:
//
//   * the raw stream is Philox4x64-10 (Salmon et al., "Parallel random numbers:
//     as easy as 1, 2, 3"), counter-based, so any raw position is directly
//     addressable: raw draw d is word d % 4 of block counter d / 4 + 1 (numpy
//     increments the counter before producing a block);
//   * each normal is decoded by numpy's own ziggurat, random_standard_normal()
//     from numpy/random/lib/libnpyrandom.a (linked statically), fed through
//     numpy's bitgen_t interface -- so the fast path, the tail and the wedge
//     rejection (with the platform libm exp/log1p numpy uses) are numpy's;
//   * a normal consumes one raw draw ~99.3% of the time and more on the slow
//     paths, so normal k's raw position is only known sequentially.  Threads
//     decode contiguous raw chunks speculatively from the chunk start; the true
//     start of chunk t+1 is where chunk t's last normal ends, and because the
//     decode re-synchronises within a few draws, each chunk is fixed up by
//     re-decoding only up to the point where the two decode paths meet.
#include <stdint.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

extern "C" {
// numpy/random/bitgen.h
typedef struct bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
} bitgen_t;
double random_standard_normal(bitgen_t* bitgen_state);
}

namespace rq {
namespace {

struct Philox {
  uint64_t k0, k1;
  uint64_t pos = 0;              // next raw draw
  uint64_t blk = ~0ull;          // block held in buf
  uint64_t buf[4];
};

inline void philox_block(uint64_t block, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c0 = block + 1, c1 = c0 == 0 ? 1 : 0, c2 = 0, c3 = 0;   // 256-bit counter block + 1
  for (int r = 0; r < 10; ++r) {
    const unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ull * c0;
    const unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ull * c2;
    const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

uint64_t next64(void* st) {
  Philox* s = (Philox*)st;
  const uint64_t b = s->pos >> 2;
  if (b != s->blk) {
    philox_block(b, s->k0, s->k1, s->buf);
    s->blk = b;
  }
  return s->buf[s->pos++ & 3];
}
uint32_t next32(void* st) { return (uint32_t)(next64(st) >> 32); }  // unused by the ziggurat
double nextd(void* st) { return (double)(next64(st) >> 11) * (1.0 / 9007199254740992.0); }

struct Decoder {
  Philox ph;
  bitgen_t bg;
  Decoder(uint64_t k0, uint64_t k1) {
    ph.k0 = k0;
    ph.k1 = k1;
    bg.state = &ph;
    bg.next_uint64 = next64;
    bg.next_uint32 = next32;
    bg.next_double = nextd;
    bg.next_raw = next64;
  }
  // the normal whose first raw draw is `at`; returns the position after it
  uint64_t decode(uint64_t at, double& v) {
    ph.pos = at;
    v = random_standard_normal(&bg);
    return ph.pos;
  }
};

// one thread's decode (cache-line aligned: adjacent chunks are written concurrently)
struct alignas(128) Chunk {
  std::vector<uint64_t> start;   // raw start of each decoded normal
  std::vector<double> val;
  size_t n = 0;
  uint64_t end = 0;              // raw position after the last decoded normal
  void push(uint64_t p, double v) {
    if (n == start.size()) {
      start.resize(2 * n + 64);
      val.resize(2 * n + 64);
    }
    start[n] = p;
    val[n] = v;
    ++n;
  }
};

// decode normals starting at raw `from` until the next start is >= `until`
void decode_range(Decoder& d, uint64_t from, uint64_t until, Chunk& c) {
  c.n = 0;
  if (c.start.size() < until - from + 16) {
    c.start.resize(until - from + 16);
    c.val.resize(until - from + 16);
  }
  uint64_t* st = c.start.data();
  double* vv = c.val.data();
  size_t k = 0;
  uint64_t p = from;
  while (p < until) {   // at most until - from normals: each consumes >= 1 draw
    st[k] = p;
    p = d.decode(p, vv[k]);
    ++k;
  }
  c.n = k;
  c.end = p;
}

// Fork-join worker pool kept across calls: creating 15 threads per call cost
// ~0.4 ms of a ~1.8 ms cfg2 draw.  run(T, f) executes f(0..T-1), f(0) on the
// caller.
class Pool {
 public:
  void run(int T, const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> lk(m_);
    while ((int)th_.size() < T - 1) {
      const int idx = (int)th_.size() + 1;
      th_.emplace_back([this, idx] { worker(idx); });
      th_.back().detach();
    }
    job_ = &f;
    active_ = T;
    pending_ = T - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    f(0);
    lk.lock();
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void worker(int idx) {
    int seen = 0;
    std::unique_lock<std::mutex> lk(m_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (idx >= active_) continue;
      const std::function<void(int)>* f = job_;
      lk.unlock();
      (*f)(idx);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::mutex m_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> th_;
  const std::function<void(int)>* job_ = nullptr;
  int gen_ = 0, active_ = 0, pending_ = 0;
};

Pool& pool() {
  static Pool* p = new Pool();   // never destroyed: detached workers outlive static destructors
  return *p;
}

}  // namespace
}  // namespace rq

// count normals of Philox(key = k0 + 2^64 k1).standard_normal starting at raw
// draw `raw`, into out[0..count); *raw_end = raw position of the next normal
extern "C" int rq_omega_fill(uint64_t k0, uint64_t k1, uint64_t raw, double* out, int64_t count,
                             int threads, uint64_t* raw_end) {
  using namespace rq;
  if (count < 0 || (count > 0 && out == nullptr) || raw_end == nullptr) return -1;
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(threads, count / 16384));
  if (T == 1) {
    Decoder d(k0, k1);
    uint64_t p = raw;
    for (int64_t i = 0; i < count; ++i) p = d.decode(p, out[i]);
    *raw_end = p;
    return 0;
  }
  // raw draws per normal ~1.0071; chunk t covers [raw + t D, raw + (t+1) D)
  const uint64_t D = (uint64_t)((double)count * 1.0071 / T) + 64;
  // chunk buffers persist across calls (first-touch page faults of fresh
  // per-call buffers serialise the threads in the kernel)
  static std::mutex mu;
  static std::vector<Chunk> pool_chunks;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)pool_chunks.size() < T) pool_chunks.resize(T);
  std::vector<Chunk>& ch = pool_chunks;
  pool().run(T, [&](int t) {
    Decoder d(k0, k1);
    decode_range(d, raw + t * D, raw + (t + 1) * D, ch[t]);
  });
  // fix-up: chunk t's true first start is chunk t-1's end
  Decoder d(k0, k1);
  std::vector<size_t> first(T, 0);
  for (int t = 1; t < T; ++t) {
    const uint64_t e = ch[t - 1].end;
    Chunk& c = ch[t];
    const uint64_t* cs = c.start.data();
    const size_t k0i = (size_t)(std::lower_bound(cs, cs + c.n, e) - cs);
    if (k0i < c.n && cs[k0i] == e) {
      first[t] = k0i;
      continue;
    }
    // re-decode from e until the path meets a recorded start (or passes the chunk)
    Chunk fix;
    uint64_t p = e;
    double v;
    size_t k = k0i;
    while (true) {
      while (k < c.n && cs[k] < p) ++k;
      if (k < c.n && cs[k] == p) break;
      if (p >= raw + (t + 1) * D) { k = c.n; break; }
      const uint64_t q = d.decode(p, v);
      fix.push(p, v);
      p = q;
    }
    for (size_t i = k; i < c.n; ++i) fix.push(c.start[i], c.val[i]);
    fix.end = k < c.n ? c.end : p;
    c = std::move(fix);
    first[t] = 0;
  }
  // concatenate (in parallel); extend sequentially if the chunks fell short
  std::vector<int64_t> off(T + 1, 0), take(T, 0);
  int64_t n = 0;
  int tl = -1;
  for (int t = 0; t < T && n < count; ++t) {
    const size_t avail = ch[t].n - first[t];
    take[t] = std::min<int64_t>((int64_t)avail, count - n);
    off[t] = n;
    n += take[t];
    tl = t;
  }
  pool().run(T, [&](int t) {
    if (take[t] > 0)
      std::memcpy(out + off[t], ch[t].val.data() + first[t], (size_t)take[t] * sizeof(double));
  });
  if (n == count && tl >= 0) {
    const size_t last = first[tl] + (size_t)take[tl];   // index after the count-th normal
    *raw_end = last < ch[tl].n ? ch[tl].start[last] : ch[tl].end;
    return 0;
  }
  uint64_t p = ch[T - 1].end;
  for (; n < count; ++n) p = d.decode(p, out[n]);
  *raw_end = p;
  return 0;
}
