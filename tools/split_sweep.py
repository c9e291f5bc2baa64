"""Per-block phase durations of one cfg2 factorization under different SM
splits.  For every block: the panel phase (panel start -> first small GEMM,
i.e. max(fast panel, inner H)) and the select phase (trailing update start ->
next swap, i.e. max(select, update)).
Usage: python tools/split_sweep.py out.jsonl opt=v1,v2,... [opt2=...]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1509_06820_b200 as P
from paper_1509_06820_b200 import _abi

cfg = bench.CONFIGS[os.environ.get("CFG", "cfg2")]
dev = torch.device("cuda", 0)
A = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
lib, h = _abi.load_library(), _abi.handle(0)
out = open(sys.argv[1], "w")


def trace():
    _abi.check(lib.rq_set_option(h, b"profile_trace", 1))
    _abi.check(lib.rq_profile_enable(h, 1))
    _abi.check(lib.rq_profile_reset(h))
    bench.run_ours(P, cfg, A, None)
    torch.cuda.synchronize()
    _abi.check(lib.rq_profile_enable(h, 0))
    cap = 20000
    cat, st, en, cnt = (C.c_int32 * cap)(), (C.c_double * cap)(), (C.c_double * cap)(), C.c_int64()
    _abi.check(lib.rq_profile_trace(h, cap, cat, st, en, C.byref(cnt)))
    n = min(cnt.value, cap)
    _abi.check(lib.rq_set_option(h, b"profile_trace", 0))
    return sorted((st[i], en[i], _abi.PROF_NAMES[cat[i]]) for i in range(n))


def phases(recs):
    sw = [i for i, x in enumerate(recs) if x[2] == "swap"]
    res = []
    for b in range(len(sw) - 1):
        seg = recs[sw[b]:sw[b + 1] + 1]
        names = [x[2] for x in seg]
        try:
            p0 = next(x[0] for x in seg if x[2] == "panel")
            g0 = next(x[0] for x in seg if x[2] == "small_gemm")
            u0 = next(x[0] for x in seg if x[2] == "update")
        except StopIteration:
            res.append(None)
            continue
        res.append({"panel": round(1e3 * (g0 - p0), 1), "select": round(1e3 * (seg[-1][0] - u0), 1),
                    "cad": round(1e3 * (seg[-1][0] - seg[0][0]), 1), "n": len(names)})
    return res


settings = [[]]
for arg in sys.argv[2:]:
    k, vs = arg.split("=")
    settings = [s + [(k, int(v))] for s in settings for v in vs.split(",")]
for s in settings:
    for k, v in s:
        _abi.check(lib.rq_set_option(h, k.encode(), v))
    bench.run_ours(P, cfg, A, None)
    torch.cuda.synchronize()
    t = trace()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bench.run_ours(P, cfg, A, None); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    out.write(json.dumps({"opts": dict(s), "ms": round(min(ms), 2), "blocks": phases(t)}) + "\n")
    out.flush()
    print(json.dumps({"opts": dict(s), "ms": round(min(ms), 2)}), flush=True)
