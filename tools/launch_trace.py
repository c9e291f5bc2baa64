"""Device-timeline trace of one factorization: per-family busy time and the
idle gaps before each family's launches.  Usage: python tools/launch_trace.py cfg2"""
import ctypes as C
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1509_06820_b200 as P
from paper_1509_06820_b200 import _abi

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
dev = torch.device("cuda", 0)
A = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
lib, h = _abi.load_library(), _abi.handle(0)
for kv in sys.argv[2:]:   # option overrides, name=value
    k, v = kv.split("=")
    _abi.check(lib.rq_set_option(h, k.encode(), int(v)))
bench.run_ours(P, cfg, A, None)
torch.cuda.synchronize()
_abi.check(lib.rq_set_option(h, b"profile_trace", 1))
_abi.check(lib.rq_profile_enable(h, 1))
_abi.check(lib.rq_profile_reset(h))
bench.run_ours(P, cfg, A, None)
torch.cuda.synchronize()
_abi.check(lib.rq_profile_enable(h, 0))
cap = 20000
cat = (C.c_int32 * cap)()
st = (C.c_double * cap)()
en = (C.c_double * cap)()
cnt = C.c_int64()
_abi.check(lib.rq_profile_trace(h, cap, cat, st, en, C.byref(cnt)))
n = min(cnt.value, cap)
recs = sorted((st[i], en[i], _abi.PROF_NAMES[cat[i]]) for i in range(n))
busy = defaultdict(float)
gap_before = defaultdict(float)
gap_after = defaultdict(float)
big = []
prev_end, prev_name = recs[0][0], None
for s0, e0, nm in recs:
    busy[nm] += e0 - s0
    g = max(0.0, s0 - prev_end)
    gap_before[nm] += g
    if prev_name:
        gap_after[prev_name] += g
    if g > 0.05:
        big.append((round(g, 3), prev_name, nm, round(s0, 2)))
    prev_end, prev_name = max(prev_end, e0), nm
span = recs[-1][1] - recs[0][0]
print(json.dumps({"launches": n, "span_ms": round(span, 2), "busy_ms": round(sum(busy.values()), 2),
                  "idle_ms": round(span - sum(busy.values()), 2)}))
print(json.dumps({"busy": {k: round(v, 2) for k, v in busy.items()}}))
cnt_f = defaultdict(int)
for _, _, nm in recs:
    cnt_f[nm] += 1
print(json.dumps({"mean_us": {k: round(1e3 * busy[k] / cnt_f[k], 1) for k in busy},
                  "count": dict(cnt_f)}))
print(json.dumps({"gap_before": {k: round(v, 2) for k, v in gap_before.items()}}))
print(json.dumps({"gap_after": {k: round(v, 2) for k, v in gap_after.items()}}))
print(json.dumps({"largest_gaps": sorted(big, reverse=True)[:15]}))
# concurrency: time where a select interval overlaps an update interval
sel = [(a, b) for a, b, nm in recs if nm == "select"]
upd = [(a, b) for a, b, nm in recs if nm == "update"]
ov = 0.0
j = 0
for a, b in sel:
    for c, d in upd:
        ov += max(0.0, min(b, d) - max(a, c))
print(json.dumps({"select_update_overlap_ms": round(ov, 2), "select_ms": round(sum(b - a for a, b in sel), 2),
                  "update_ms": round(sum(b - a for a, b in upd), 2)}))
pairs = []
for a, b in sel[:200]:
    best = max(((min(b, d) - max(a, c)), c, d) for c, d in upd) if upd else (0, 0, 0)
    pairs.append((round(a, 3), round(b - a, 3), round(best[0], 3), round(best[2] - best[1], 3)))
print(json.dumps({"first_selects(start,dur,overlap,upd_dur)": pairs[:12]}))
# exposed time per family: intervals where it is the only family running
ev = []
for a, b, nm in recs:
    ev.append((a, 1, nm)); ev.append((b, -1, nm))
ev.sort()
active = {}
exposed = defaultdict(float)
idle = 0.0
last = ev[0][0]
for t, d, nm in ev:
    run = [k for k, v in active.items() if v > 0]
    if len(run) == 1:
        exposed[run[0]] += t - last
    elif not run:
        idle += t - last
    last = t
    active[nm] = active.get(nm, 0) + d
print(json.dumps({"exposed_ms": {k: round(v, 2) for k, v in sorted(exposed.items(), key=lambda x: -x[1])},
                  "idle_ms": round(idle, 2)}))
if os.environ.get("TRACE_DUMP"):
    with open(os.environ["TRACE_DUMP"], "w") as f:
        json.dump([(round(a, 4), round(b, 4), nm) for a, b, nm in recs], f)
_abi.check(lib.rq_set_option(h, b"profile_trace", 0))
