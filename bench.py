#!/usr/bin/env python
"""Benchmark: blocked RQRCP FP64 GFLOP/s on B200 (BASELINE.json metric).

Default workload = BASELINE config 2: full RQRCP of an 8192 x 8192 FP64
matrix A = U diag(sigma) V^T, sigma_i = 10^(-12 i / 8191), b = 64, p = 8, on
one B200.  A "step" is one complete factorization (all 128 blocks) through the
public API with A already resident in HBM.  GFLOP/s counts standard
Householder QR flops (4n^3/3 full, 4kmn - 2k^2(m+n) + 4k^3/3 truncated).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1|cfg2|cfg3|cfg4|cfg5]

Prints ONE JSON line on rank 0.  Under torchrun (N > 1) the matrix is sharded
column-block-cyclically over the ranks and factored by the NCCL driver
(paper_1509_06820_b200/parallel.py; strong scaling), timed between barriers
with CUDA events, max over ranks.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(driver="rqrcp", m=1000, n=1000, k=None, block=32, padding=8, kind="gauss",
                 desc="RQRCP full, 1000x1000 N(0,1), b=32, p=8"),
    "cfg2": dict(driver="rqrcp", m=8192, n=8192, k=None, block=64, padding=8, kind="geom12",
                 desc="RQRCP full, 8192x8192 A=U diag(10^(-12 i/8191)) V^T, b=64, p=8"),
    "cfg3": dict(driver="trqrcp", m=16384, n=16384, k=512, block=64, padding=8, kind="lowrank600",
                 desc="TRQRCP k=512, 16384^2 = G(16384x600) G(600x16384) + 1e-6 N(0,1), b=64, p=8"),
    "cfg4": dict(driver="tuxv", m=20000, n=12000, k=256, block=32, padding=8, kind="inv_sq",
                 desc="TUXV k=256, 20000x12000, sigma_i = 1/(1+i)^2, b=32, p=8"),
    "cfg5": dict(driver="rqrcp", m=32768, n=32768, k=None, block=128, padding=8, kind="gauss",
                 desc="RQRCP full, 32768x32768 N(0,1), b=128, p=8"),
}
# bounded CPU sample of the same workload (n of the n x n instance of the same
# recipe) for the oracle: one size for both cpu_baseline and --impl reference,
# each run a few seconds on the box's host cores
CPU_SAMPLE = {"cfg1": 1000, "cfg2": 2048, "cfg3": 4096, "cfg4": 2500, "cfg5": 2048}


def std_flops(cfg, m=None, n=None, k=None):
    m = m or cfg["m"]
    n = n or cfg["n"]
    if cfg["driver"] == "rqrcp":
        k = min(m, n)
        if m == n:
            return 4.0 * n ** 3 / 3.0
        return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0 if m >= n else 2.0 * n * m * m - 2.0 * m ** 3 / 3.0
    k = k or cfg["k"]
    return 4.0 * k * m * n - 2.0 * k * k * (m + n) + 4.0 * k ** 3 / 3.0


# ------------------------------------------------------------------ inputs

def host_matrix(kind, m, n, seed=0):
    """Seeded CPU recipe; used for the CPU oracle samples."""
    rng = np.random.default_rng(seed)
    if kind == "gauss":
        return rng.standard_normal((m, n))
    if kind == "geom12":
        U = np.linalg.qr(rng.standard_normal((n, n)))[0]
        V = np.linalg.qr(rng.standard_normal((n, n)))[0]
        s = 10.0 ** (-12.0 * np.arange(n) / (n - 1))
        return np.asfortranarray((U * s) @ V.T)
    if kind == "lowrank600":
        r = min(600, m // 4)
        return rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) \
            + 1e-6 * rng.standard_normal((m, n))
    if kind == "inv_sq":
        U = np.linalg.qr(rng.standard_normal((m, n)))[0]
        V = np.linalg.qr(rng.standard_normal((n, n)))[0]
        s = 1.0 / (1.0 + np.arange(n)) ** 2
        return np.asfortranarray((U * s) @ V.T)
    raise ValueError(kind)


def device_matrix(kind, m, n, device, seed=0):
    """Same recipe with the seeded Gaussians drawn on the host (numpy PCG64,
    bit-identical to the CPU recipe) and the QR / products done on the GPU
    through torch (input generation only, outside every timed region)."""
    import torch
    from paper_1509_06820_b200.device import fmat
    rng = np.random.default_rng(seed)

    def gauss(r, c):
        if r * c > (1 << 29):  # > 4 GiB: draw on the device instead
            g = torch.Generator(device=device).manual_seed(seed + r + c)
            return torch.randn((c, r), dtype=torch.float64, device=device, generator=g).t()
        return torch.from_numpy(rng.standard_normal((r, c))).to(device)

    if kind == "gauss":
        G = gauss(m, n)
        A = fmat(m, n, device)
        A.copy_(G)
        return A
    if kind in ("geom12", "inv_sq"):
        U = torch.linalg.qr(gauss(m, n))[0]
        V = torch.linalg.qr(gauss(n, n))[0]
        i = torch.arange(n, dtype=torch.float64, device=device)
        s = 10.0 ** (-12.0 * i / (n - 1)) if kind == "geom12" else 1.0 / (1.0 + i) ** 2
        A = fmat(m, n, device)
        A.copy_((U * s) @ V.T)
        return A
    if kind == "lowrank600":
        G1 = gauss(m, 600)
        G2 = gauss(600, n)
        G3 = gauss(m, n)
        A = fmat(m, n, device)
        A.copy_(G1 @ G2 + 1e-6 * G3)
        return A
    raise ValueError(kind)


def recipe_matrix(name, device):
    """The configuration's A from the exact SURVEY.md §8(d) numpy recipe
    (tests/golden/recipes.py, the bytes the parity goldens were generated
    from), built on the host and uploaded: the bench and the full-size
    parity tests factor the same matrix.  Input generation, outside every
    timed region."""
    import torch
    from paper_1509_06820_b200.device import fmat
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import recipes
    Ah = recipes.build_as_golden(name)
    A = fmat(Ah.shape[0], Ah.shape[1], device)
    A.copy_(torch.from_numpy(Ah))
    return A


# ------------------------------------------------------------------ helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) must not overlap the timed
            # region: wait for its first sample, then drop it
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def window(self, t0, t1):
        """Summary of the samples taken between host times t0 and t1 (the
        sampler runs across the whole bench, so its start-up and the NVML
        queries' first costs fall in the warm-up, not in a timed pass)."""
        lines = list(self.lines)
        pad = 0.0
        win = [(t, ln) for t, ln in lines if t0 <= t <= t1]
        while len(win) < 3 and pad < 0.2:   # a short pass: widen to the nearest samples
            pad += 0.04
            win = [(t, ln) for t, ln in lines if t0 - pad <= t <= t1 + pad]
        out = self.summary(win)
        if pad:
            out["window_padded_ms"] = round(1e3 * pad)
        return out

    def summary(self, lines=None):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in (self.lines if lines is None else lines):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak():
    """Measured FP64 DMMA / FFMA64 peak (MEASURED_PEAKS.json has no FP64 entry)."""
    exe = os.path.join(ROOT, "paper_1509_06820_b200", "fp64_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception:
        return None


def cpu_run(cfg_name, n_sample):
    """Time the CPU oracle (oracle/port.py, the reference algorithm restated in
    numpy/OpenBLAS) on a bounded sample of the workload; all host cores."""
    from threadpoolctl import threadpool_limits
    from oracle import port
    cfg = CONFIGS[cfg_name]
    m = n = n_sample
    if cfg["kind"] == "inv_sq":
        m = int(n_sample * cfg["m"] / cfg["n"])
    A = host_matrix(cfg["kind"], m, n)
    cores = os.cpu_count() or 1
    b, p = cfg["block"], cfg["padding"]
    k = None if cfg["k"] is None else min(cfg["k"], n // 4)
    with threadpool_limits(cores):
        t0 = time.perf_counter()
        if cfg["driver"] == "rqrcp":
            port.rqrcp(A, None, b, p, 0)
        elif cfg["driver"] == "trqrcp":
            port.trqrcp(A, k, b, p, 0)
        else:
            port.tuxv(A, k, b, p, 0)
        dt = time.perf_counter() - t0
    sub = dict(cfg, m=m, n=n, k=k)
    return std_flops(sub, m, n, k) / dt / 1e9, dt, cores, m, n, k


def run_ours(P, cfg, A, extra_cfg):
    config = P.RandomizedConfig(block=cfg["block"], padding=cfg["padding"], seed=0)
    if cfg["driver"] == "rqrcp":
        return P.rqrcp(A, cfg["k"], config)
    if cfg["driver"] == "trqrcp":
        return P.trqrcp(A, cfg["k"], config)
    return P.tuxv(A, cfg["k"], config)


def result_bytes(f, cfg):
    tot = 0
    for name in ("R", "trailing", "U", "V", "X"):
        t = getattr(f, name, None)
        if t is not None:
            tot += t.nbytes
    refl = getattr(f, "reflectors", None)
    if refl is not None:
        for t in (refl.Y, refl.tau, refl.W):
            if t is not None:
                tot += t.nbytes
    perm = getattr(f, "perm", None)
    if perm is not None:
        tot += np.asarray(perm.forward).nbytes
    return tot


# ------------------------------------------------------------------ main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the column-block-cyclic driver even at N = 1 (tests the N > 1 path)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return main_reference(args, cfg, rank)

    import torch
    import torch.distributed as dist
    import paper_1509_06820_b200 as P
    from paper_1509_06820_b200 import _abi
    import ctypes as C

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_sharded:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    peak = fp64_peak() if rank == 0 else None
    A = recipe_matrix(args.config, dev)
    torch.cuda.synchronize(dev)
    lib = _abi.load_library()
    h = _abi.handle(local)
    # diagnostics: RQ_OPTIONS="name=value,..." sets library options (rq_set_option)
    for kv in filter(None, os.environ.get("RQ_OPTIONS", "").split(",")):
        k, v = kv.split("=")
        _abi.check(lib.rq_set_option(h, k.strip().encode(), int(v)))

    sharded = world > 1 or args.force_sharded
    if sharded:
        # column-block-cyclic shards of ONE matrix over the ranks (strong scaling)
        from paper_1509_06820_b200.parallel import BlockCyclic, rqrcp_sharded
        layout = BlockCyclic(cfg["n"], cfg["block"], world)
        idx = torch.as_tensor(layout.positions(rank), device=dev)
        from paper_1509_06820_b200.device import fmat
        A_loc = fmat(cfg["m"], int(idx.numel()), dev)
        A_loc.copy_(A[:, idx])
        del A
        torch.cuda.empty_cache()
        if cfg["driver"] == "tuxv":
            raise SystemExit("multi-GPU bench: TUXV is not sharded (RQRCP and TRQRCP are)")
        from paper_1509_06820_b200.parallel import trqrcp_sharded
        cfgP = P.RandomizedConfig(block=cfg["block"], padding=cfg["padding"], seed=0)

        def step(P_, cfg_, A_, _x):
            if cfg_["driver"] == "trqrcp":
                return trqrcp_sharded(A_loc, cfg_["m"], cfg_["n"], cfg_["k"], cfgP, gather=False)
            return rqrcp_sharded(A_loc, cfg_["m"], cfg_["n"], cfg_["k"], cfgP, gather_r=False)
        A = None
    else:
        step = run_ours
    # clocks are sampled by one nvidia-smi process for the whole run (started
    # before the warm-up); each timed pass reports the samples of its window
    sampler = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        f = step(P, cfg, A, None)
    barrier()
    stream = torch.cuda.current_stream(dev)

    def timed_pass(profile):
        """K steps bracketed by barrier + synchronize, CUDA events on the
        launching stream; with `profile` the library also records events
        around every kernel launch (per-family durations for the roofline)."""
        _abi.check(lib.rq_profile_reset(h))
        _abi.check(lib.rq_profile_enable(h, 1 if profile else 0))
        # no Python garbage collection pauses between the K calls (a gen-2
        # pass with torch loaded idles the GPU for tens of ms)
        gc.collect()
        gc.disable()
        l0 = lib.rq_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        t0 = time.time()
        # NVTX range: `ncu --nvtx --nvtx-include timed/` lists exactly the
        # headline pass's launches
        torch.cuda.nvtx.range_push("timed" if not profile else "profiled")
        e0.record(stream)
        marks = []   # per-step events (idle gaps between calls show up here)
        f_ = None
        for _ in range(args.steps):
            f_ = None   # the previous result is released before the next call
            f_ = step(P, cfg, A, None)
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record(stream)
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
        t1 = time.time()
        _abi.check(lib.rq_profile_enable(h, 0))
        gc.enable()
        steps_ms = [round(a_.elapsed_time(b_), 3) for a_, b_ in zip([e0] + marks[:-1], marks)]
        timed_pass.steps_ms = steps_ms
        return f_, e0.elapsed_time(e1), lib.rq_launch_count() - l0, sampler.window(t0, t1)

    # headline pass without per-launch events, then the same K steps again
    # with them (kernel shares and the roofline's per-launch durations)
    # the warm-up's last result would otherwise stay alive through the timed
    # pass: three result sets at once make the caching allocator grow (cudaMalloc)
    # inside the second timed call
    f = None
    f, ms, launches, clk = timed_pass(False)
    f = None
    steps_ms = timed_pass.steps_ms
    f, ms_prof, _, clk_prof = timed_pass(True)
    sampler.__exit__(None, None, None)
    n_cat = len(_abi.PROF_NAMES)
    L = (C.c_int64 * n_cat)()
    MS = (C.c_double * n_cat)()
    FL = (C.c_double * n_cat)()
    BY = (C.c_double * n_cat)()
    _abi.check(lib.rq_profile_read(h, L, MS, FL, BY))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    flops_step = std_flops(cfg)
    # replicas: every rank factors its own matrix; sharded: one matrix over all ranks
    value = flops_step * (1 if sharded else world) / (ms_step * 1e-3) / 1e9
    kernels = {}
    for i, nm in enumerate(_abi.PROF_NAMES):
        if L[i]:
            kernels[nm] = {"launches_per_step": L[i] / args.steps, "ms_per_step": MS[i] / args.steps,
                           "share": MS[i] / max(ms_prof, 1e-9),
                           "tflops": FL[i] / max(MS[i], 1e-9) / 1e9 if FL[i] else None,
                           "gbs": BY[i] / max(MS[i], 1e-9) / 1e6 if BY[i] else None}
    gemm_fams = [nm for nm in ("update", "inner", "sketch", "small_gemm") if nm in kernels]
    dom = max(gemm_fams, key=lambda nm: kernels[nm]["ms_per_step"]) if gemm_fams else None
    roofline = None
    if dom is not None:
        i = _abi.PROF_NAMES.index(dom)
        ach = FL[i] / (MS[i] * 1e-3) / 1e12
        pk = peak["dmma_f64_tflops"] if peak else 37.2
        kname = {"update": "rank_update_grouped_kernel (C -= Y X, K = b; TMA, one CTA/SM of "
                           "three 4-warp groups on 64x64 tiles, C tile prefetched by TMA)",
                 "inner": "tc_tma_kernel (G = Y^T C, TMA-fed, split-K)",
                 "sketch": "tc_tma_kernel (B = Omega A, TMA-fed)",
                 "small_gemm": "tc_tma_kernel / block_finish_kernel (small products)"}.get(dom, dom)
        roofline = {"bound": "tensor", "kernel": kname, "achieved": ach,
                    "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                    "traffic": traffic_from_profiles(dom),
                    "peak_source": ("measured DMMA.8x8x4 microbenchmark in this run "
                                    "(MEASURED_PEAKS.json has no FP64 figure)") if peak else
                    "boost-clock derivation 148 SM x 128 flop/clk x 1.965 GHz",
                    "algorithmic_flops_per_launch": FL[i] / max(L[i], 1),
                    "avg_launch_us": MS[i] * 1e3 / max(L[i], 1),
                    "share": kernels[dom]["share"]}
        if dom == "update":
            roofline["note"] = ("the trailing update runs beside the next block's pivot selection "
                                "on the SMs that leaves free (cfg2: 104 of 148, 68 from block ~56 "
                                "on; cfg5: ~90-105); `achieved` is per launch on that share, "
                                "`peak` is the whole chip's")
    res_counters = f.counters
    if sharded:
        from paper_1509_06820_b200.factorization import OpCounters
        res_counters = OpCounters(gemm_flops=f.counters["gemm_flops"],
                                  level2_flops=f.counters["level2_flops"],
                                  resamples=f.counters["resamples"])

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e and rank == 0 and not sharded:
        Ah = torch.empty((cfg["n"], cfg["m"]), dtype=torch.float64).pin_memory().t()
        Ah.copy_(A)
        Ahost = Ah.numpy()
        # W warm-up calls of the host path, as for the device leg (the first
        # calls also size torch's caching pinned-host allocator for results)
        for _ in range(max(args.warmup, 1)):
            f = run_ours(P, cfg, Ahost, None)
        d2h = result_bytes(f, cfg)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            f = run_ours(P, cfg, Ahost, None)
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": flops_step / dt / 1e9, "unit": "GFLOP/s", "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": int(8 * cfg["m"] * cfg["n"]), "d2h_bytes_per_step": int(d2h),
               "path": "rqrcp/trqrcp/tuxv(numpy host array in pinned memory) -> numpy results"}
        del Ah, Ahost

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        gf, dt, cores, m, n, k = cpu_run(args.config, CPU_SAMPLE[args.config])
        cpu = {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "port",
               "sample": f"oracle/port.py {cfg['driver']} on the {m}x{n} instance of the same "
                         f"recipe ({cfg['kind']}), b={cfg['block']}, p={cfg['padding']}"
                         + (f", k={k}" if k else "") + f", 1 run, {dt:.2f} s, numpy/OpenBLAS "
                         f"with {cores} threads"}

    if rank == 0:
        line = {
            "metric": "RQRCP/TRQRCP FP64 GFLOP/s (standard QR flop count), % of FP64 peak",
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_of(args.config, world, sharded),
            "pct_fp64_peak": (value / world / 1e3) / (peak["dmma_f64_tflops"] if peak else 37.2),
            "pct_fp64_peak_note": "per GPU, of the measured DMMA peak",
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "kernels": kernels,
            "steps_ms": steps_ms,
            "profiled_pass": {"ms_per_step": ms_prof / args.steps, "clocks": clk_prof,
                              "note": "same K steps re-run with CUDA events around every "
                                      "library launch; `kernels` and `roofline` come from it"},
            "counters": {"gemm_flops": res_counters.gemm_flops,
                         "level2_flops": res_counters.level2_flops,
                         "resamples": res_counters.resamples},
            "fp64_peak": peak,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def config_of(name, world, sharded):
    cfg = CONFIGS[name]
    return {"workload": name, "desc": cfg["desc"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"],
            "block": cfg["block"], "padding": cfg["padding"],
            "parallelism": (f"column-block-cyclic x{world} (NCCL)" if sharded else "single GPU"),
            "l2": "inputs larger than L2 (A is 8*m*n bytes)",
            "input": "exact SURVEY 8(d) numpy recipe (tests/golden/recipes.py), the bytes of "
                     "the reference-generated parity goldens"}


def traffic_from_profiles(family):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary (profiles/latest_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "latest_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(family)
    except Exception:
        return None


def main_reference(args, cfg, rank):
    """The reference's own CPU algorithm (oracle/port.py restatement; the
    reference is Python, so there is no compiled oracle/_ref) on the host
    cores, one bounded sample of the workload per step."""
    if rank != 0:
        return 0
    n_s = CPU_SAMPLE[args.config]
    for _ in range(args.warmup):
        cpu_run(args.config, n_s)
    vals, times = [], []
    for _ in range(args.steps):
        gf, dt, cores, m, n, k = cpu_run(args.config, n_s)
        vals.append(gf)
        times.append(dt)
    value = float(statistics.median(vals))
    sample = (f"oracle/port.py {cfg['driver']} on the {m}x{n} instance of the {args.config} recipe "
              f"({cfg['kind']}), b={cfg['block']}, p={cfg['padding']}" + (f", k={k}" if k else ""))
    line = {
        "metric": "RQRCP/TRQRCP FP64 GFLOP/s (standard QR flop count), % of FP64 peak",
        "impl": "reference", "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_of(args.config, 1, False),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
