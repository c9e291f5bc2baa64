"""Full-size parity of one config against the CPU oracle on the same box:
the GPU factorization (native driver) and oracle/port.py (the reference's
numpy algorithm) on the same A bytes and seed.  Reports identical pivots,
||R - R_oracle|| / ||R_oracle||, the residual of the GPU factorization on a
column sample, and the counters.
Usage: python tools/full_parity.py cfg2 out.json [m=.. n=.. block=..]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1509_06820_b200 as P
from oracle import port

name = sys.argv[1]
cfg = dict(bench.CONFIGS[name])
for kv in sys.argv[3:]:   # overrides, e.g. m=8192 n=8192 block=32
    k_, v_ = kv.split("=")
    cfg[k_] = v_ if k_ in ("driver", "kind") else int(v_)
    name += f" {k_}={v_}"
dev = torch.device("cuda", 0)
A_d = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
A = A_d.cpu().numpy()
A = np.asfortranarray(A)
conf = P.RandomizedConfig(block=cfg["block"], padding=cfg["padding"], seed=0)
drv = cfg["driver"]
run_gpu = {"rqrcp": lambda: P.rqrcp(A_d, cfg["k"], conf), "trqrcp": lambda: P.trqrcp(A_d, cfg["k"], conf),
           "tuxv": lambda: P.tuxv(A_d, cfg["k"], conf),
           "rsrqrcp": lambda: P.rsrqrcp(A_d, cfg["k"], conf),
           "ssrqrcp": lambda: P.ssrqrcp(A_d, cfg["k"], conf)}[drv]
run_cpu = {"rqrcp": lambda: port.rqrcp(A, cfg["k"], cfg["block"], cfg["padding"], 0),
           "rsrqrcp": lambda: port.rsrqrcp(A, cfg["k"], cfg["block"], cfg["padding"], 0),
           "ssrqrcp": lambda: port.ssrqrcp(A, cfg["k"], cfg["block"], cfg["padding"], 0),
           "trqrcp": lambda: port.trqrcp(A, cfg["k"], cfg["block"], cfg["padding"], 0),
           "tuxv": lambda: port.tuxv(A, cfg["k"], cfg["block"], cfg["padding"], 0)}[drv]
t = time.perf_counter()
f = run_gpu()
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t
t = time.perf_counter()
o = run_cpu()
t_cpu = time.perf_counter() - t
h = lambda x: x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)
out = {"config": name, "driver": drv, "m": cfg["m"], "n": cfg["n"], "k": cfg["k"],
       "gpu_s": round(t_gpu, 3), "oracle_s": round(t_cpu, 1),
       "note": "same A bytes (generated on the device, copied to the host) and seed; oracle = "
               "oracle/port.py on this box's host cores"}
nA = np.linalg.norm(A)
if drv == "tuxv":
    s_g, s_o = h(f.singular_values()), np.asarray(o.singular_values())
    out["rank_gpu"], out["rank_oracle"] = int(f.rank), int(o.rank)
    out["sigma_max_rel_err"] = float(np.max(np.abs(s_g - s_o) / np.abs(s_o)))
    Ag = h(f.U) @ h(f.X) @ h(f.V).T
    out["approx_err_gpu"] = float(np.linalg.norm(A - Ag) / nA)
    out["approx_err_oracle"] = float(np.linalg.norm(A - o.approx()) / nA)
else:
    pf = h(f.perm.forward)
    same = pf == o.perm.forward
    kk = int(o.rank)
    out["rank_gpu"], out["rank_oracle"] = int(f.rank), kk
    out["pivots_identical"] = bool(same.all())
    out["pivots_identical_first_k"] = bool(same[:kk].all())
    out["pivot_mismatches"] = int((~same).sum())
    R = h(f.R)
    out["R_rel_err"] = float(np.linalg.norm(R - o.R) / np.linalg.norm(o.R))
    c = f.counters
    out["counters_gpu"] = [int(c.gemm_flops), int(c.level2_flops), int(c.resamples)]
    out["counters_oracle"] = [int(o.counters.gemm_flops), int(o.counters.level2_flops),
                              int(o.counters.resamples)]
    if drv in ("rqrcp", "rsrqrcp") and cfg["k"] is None:
        # residual ||A P - Q R|| on 64 sampled columns (dense Q formed on the device)
        g = np.random.default_rng(1)
        cols = np.sort(g.choice(cfg["n"], 64, replace=False))
        E = h(P.q_columns(f.reflectors.Y, f.reflectors.tau, cfg["m"]))
        out["residual_64_cols"] = float(np.linalg.norm(A[:, pf[cols]] - E @ R[:, cols])
                                        / np.linalg.norm(A[:, pf[cols]]))
    else:
        # truncation error ||A P - Q_k R_k|| / ||A|| (truncated.py quality metric)
        Qk = h(P.q_columns(f.reflectors.Y, f.reflectors.tau, kk))
        out["trunc_err_gpu"] = float(np.linalg.norm(A[:, pf] - Qk @ R) / nA)
        Qo = port.q_columns(o.Y, o.tau, kk)
        out["trunc_err_oracle"] = float(np.linalg.norm(A[:, o.perm.forward] - Qo @ o.R) / nA)
print(json.dumps(out))
json.dump(out, open(sys.argv[2], "w"), indent=1)
