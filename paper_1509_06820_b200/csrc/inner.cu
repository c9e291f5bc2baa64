// K3': the inner product of a block, H = P^T C  (b = 64 rows, K = the
// trailing rows, N = the trailing columns) -- randomized.py:170-172
// (G = Y^T C; with the fast panel the big term is P_below^T C_below, see
// driver.cu panel_overlap_inner).  Tall-skinny and compute bound (each C
// element feeds 2 b flops): 64 x 128 output tiles, eight 32 x 32 warp tiles
// (16 accumulators per warp), a 4-stage cp.async pipeline over 32-deep
// k-tiles (one barrier per 128 DMMAs per warp), and split-K into ~16 k-tile
// chunks per CTA.  Partial planes are summed in a fixed order
// (gemm_reduce_kernel): deterministic run to run.
#include "gemm.cuh"
#include "runtime.hpp"

namespace rq {

namespace {

// IM = 64: 8 warps, 2 (m) x 4 (n); IM = 32 (b = 32, cfg4): 4 warps, 1 x 4
template <int IM> struct InnerCfg {
  static constexpr int kIT = IM == 64 ? 256 : 128;
  static constexpr int kWM = IM / 32;   // warps along m
};
constexpr int kIN = 128, kIK = 32, kIS = 4;
constexpr int kILd = kIK + 4;          // As[m][k], Bs[n][k]
constexpr int kIStB = kIN * kILd;
template <int IM>
constexpr size_t inner_smem() { return (size_t)kIS * (IM * kILd + kIStB) * sizeof(double); }

struct InnerArgs {
  int64_t N, K;
  const double* P; int64_t ldp;   // K x 64, column-major
  const double* C; int64_t ldc;   // K x N, column-major
  double* out; int64_t ldo;       // 64 x N, or partial planes [split][64 x N] (ld 64)
  int64_t kchunk;                 // K rows per split (multiple of kIK)
  int tn;                         // column tiles
  const Status* st;
};

// CTA (column tile j, split z): H_z[:, tile j] = P[kz]^T C[kz, tile j].
// Not persistent: beside the fast panel the hardware scheduler moves the
// remaining CTAs onto the panel's SMs once it ends (a persistent grid sized
// to the free SMs measured slower in the driver for that reason).
template <int IM>
__global__ void __launch_bounds__(InnerCfg<IM>::kIT, 1) inner_kernel(InnerArgs a) {
  constexpr int kIM = IM, kIT = InnerCfg<IM>::kIT, kWM = InnerCfg<IM>::kWM;
  constexpr int kIStA = kIM * kILd;
  if (aborted(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                   // [kIS][kIM][kILd]
  double* Bs = As + kIS * kIStA;     // [kIS][kIN][kILd]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % kWM) * 32, wn0 = (warp / kWM) * 32;
  const int fr = lane >> 2, fk = lane & 3;
  const int j = blockIdx.x % a.tn, z = blockIdx.x / a.tn;
  const int64_t N = a.N, ldp = a.ldp, ldc = a.ldc, n0 = (int64_t)j * kIN;
  const int64_t k0 = (int64_t)z * a.kchunk;
  const int64_t k1 = k0 + a.kchunk < a.K ? k0 + a.kchunk : a.K;
  const int nkt = (int)((k1 - k0 + kIK - 1) / kIK);
  auto load = [&](int kt, int st) {
    const int64_t kb = k0 + (int64_t)kt * kIK;
#pragma unroll
    for (int q = 0; q < kIM * kIK / 2 / kIT; ++q) {   // As[m][k] <- P[kb + k, m]
      const int e = tid + q * kIT;
      const int m = e / (kIK / 2), k = 2 * (e % (kIK / 2));
      const int64_t gk = kb + k;
      const int valid = gk + 1 < k1 ? 16 : (gk < k1 ? 8 : 0);
      cp_async16(As + st * kIStA + m * kILd + k, valid ? a.P + gk + m * ldp : a.P, valid);
    }
#pragma unroll
    for (int q = 0; q < kIN * kIK / 2 / kIT; ++q) {   // Bs[n][k] <- C[kb + k, n0 + n]
      const int e = tid + q * kIT;
      const int n = e / (kIK / 2), k = 2 * (e % (kIK / 2));
      const int64_t gk = kb + k;
      const int valid = n0 + n < N ? (gk + 1 < k1 ? 16 : (gk < k1 ? 8 : 0)) : 0;
      cp_async16(Bs + st * kIStB + n * kILd + k, valid ? a.C + gk + (n0 + n) * ldc : a.C, valid);
    }
  };
#pragma unroll
  for (int s = 0; s < kIS - 1; ++s) {
    if (s < nkt) load(s, s);
    cp_async_commit();
  }
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<kIS - 2>();
    __syncthreads();   // stage kt landed; stage kt - 1 is free
    if (kt + kIS - 1 < nkt) load(kt + kIS - 1, (kt + kIS - 1) % kIS);
    cp_async_commit();
    const double* as = As + (kt % kIS) * kIStA + (wm0 + fr) * kILd;
    const double* bs = Bs + (kt % kIS) * kIStB + (wn0 + fr) * kILd;
    double af[2][4], bf[2][4];
    auto ldfrag = [&](int fb, int k4) {
#pragma unroll
      for (int x = 0; x < 4; ++x) af[fb][x] = as[x * 8 * kILd + k4 + fk];
#pragma unroll
      for (int y = 0; y < 4; ++y) bf[fb][y] = bs[y * 8 * kILd + k4 + fk];
    };
    ldfrag(0, 0);
#pragma unroll
    for (int ks = 0; ks < kIK / 4; ++ks) {
      if (ks + 1 < kIK / 4) ldfrag((ks + 1) & 1, (ks + 1) * 4);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma884(acc[x][y], af[ks & 1][x], bf[ks & 1][y]);
    }
  }
  cp_async_wait<0>();
  // acc[x][y] = rows wm0 + 8x + fr, columns wn0 + 8y + 2fk (+1)
  const bool split = a.kchunk < a.K;
  double* o = split ? a.out + (int64_t)z * (kIM * N) : a.out;
  const int64_t ldo = split ? kIM : a.ldo;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t n = n0 + wn0 + y * 8 + 2 * fk + e;
        if (n < N) o[(wm0 + x * 8 + fr) + n * ldo] = acc[x][y][e];
      }
}

}  // namespace

bool inner_gemm(Handle& h, int64_t M, int64_t N, int64_t K, const double* P, int64_t ldp,
                const double* C, int64_t ldc, double* H, int64_t ldh, cudaStream_t s,
                const Status* st, int max_ctas, int cat) {
  (void)max_ctas;
  // the second-generation GEMM is faster on every shape measured (tools/tc_bench.py)
  if (h.use_tc && N > 0 && K > 0)
    return tc_gemm(h, true, false, M, N, K, 1.0, P, ldp, C, ldc, 0.0, H, ldh, s, st, cat);
  if (!h.inner_kernel || (M != 64 && M != 32) || N <= 0 || K < 4096) return false;
  if (M == 32 && !h.inner32) return false;
  if (((uintptr_t)P & 15) || (ldp & 1) || ((uintptr_t)C & 15) || (ldc & 1)) return false;
  {
    kernel_attr((const void*)inner_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)inner_smem<64>());
                kernel_attr((const void*)inner_kernel<32>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)inner_smem<32>());
  }
  const int64_t tn = (N + kIN - 1) / kIN;
  const int64_t nkt = (K + kIK - 1) / kIK;
  // ~h.inner_ktiles k-tiles per CTA: short enough for the scheduler to
  // balance, long enough to amortise the pipeline fill
  const int64_t per = std::max(8, h.inner_ktiles);
  const int64_t sp = std::max<int64_t>(1, (nkt + per / 2) / per);
  const int64_t kc = (nkt + sp - 1) / sp * kIK;
  const int64_t spl = (K + kc - 1) / kc;
  ProfScope prof(h, cat, 2.0 * M * N * K, 8.0 * ((double)M * K + (double)K * N + (double)M * N), s);
  InnerArgs a{N, K, P, ldp, C, ldc, H, ldh, kc, (int)tn, st};
  GemmArgs g{};
  if (spl > 1) {
    a.out = (double*)h.buf("inner_partial", (size_t)spl * M * N * 8, s);
    g.M = M; g.N = N; g.K = K;
    g.C = H; g.ldc = ldh; g.alpha = 1.0; g.beta = 0.0;
    g.splits = (int)spl; g.partial = a.out; g.st = st;
  }
  if (M == 64)
    inner_kernel<64><<<(unsigned)(tn * spl), InnerCfg<64>::kIT, inner_smem<64>(), s>>>(a);
  else
    inner_kernel<32><<<(unsigned)(tn * spl), InnerCfg<32>::kIT, inner_smem<32>(), s>>>(a);
  RQ_CHECK_LAUNCH();
  count_launch();
  if (spl > 1) {
    const int64_t total = M * N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * h.num_sms);
    gemm_reduce_kernel<<<blocks, 256, 0, s>>>(g);
    RQ_CHECK_LAUNCH();
    count_launch();
  }
  return true;
}

}  // namespace rq
