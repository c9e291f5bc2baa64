"""A/B library options on one bench config in one process (device-resident
input, CUDA-event timing, interleaved repetitions).
Usage: python tools/ab_options.py cfg2 fast_panel_spec=0 fast_panel_spec=1 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1509_06820_b200 as P
from paper_1509_06820_b200 import _abi

cfg_name = sys.argv[1]
variants = [dict(kv.split("=") for kv in v.split(",")) for v in sys.argv[2:]]
cfg = bench.CONFIGS[cfg_name]
dev = torch.device("cuda", 0)
A = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
lib, h = _abi.load_library(), _abi.handle(0)


DEFAULTS = {"fast_panel": 1, "fast_panel_spec": 1, "fast_panel_max_ctas": 0, "use_rank_update": 1,
            "gemm_vec16": 1, "force_select": 0, "force_panel": 0, "select_cluster_max_cols": 1024,
            "panel_cluster_max_rows": 3072, "select_reg": 1, "select_max_ctas": 0, "overlap_select": 1, "overlap_sel_ctas": 0, "su_gemm": 1, "overlap_inner": 1, "overlap_panel_ctas": 48, "block_finish": 1, "ru_two_ctas": 0, "ru_skew_ns": 0, "ru_big": 1, "inner_kernel": 1, "inner_ktiles": 16}


def setopts(v):
    for k, x in {**DEFAULTS, **v}.items():
        _abi.check(lib.rq_set_option(h, k.encode(), int(x)))


times = {i: [] for i in range(len(variants))}
for i, v in enumerate(variants):
    setopts(v)
    bench.run_ours(P, cfg, A, None)
for rep in range(int(os.environ.get('AB_REPS', 3))):
    for i, v in enumerate(variants):
        setopts(v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = lib.rq_launch_count()
        e0.record()
        f = bench.run_ours(P, cfg, A, None)
        e1.record()
        torch.cuda.synchronize()
        times[i].append(e0.elapsed_time(e1))
        if rep == 0:
            print(json.dumps({"variant": v, "launches": lib.rq_launch_count() - l0,
                              "rank": int(f.rank), "resamples": int(f.counters.resamples)}))
for i, v in enumerate(variants):
    print(json.dumps({"variant": v, "ms": [round(t, 2) for t in times[i]], "min": round(min(times[i]), 2)}))
