"""Full-size parity of one config against the CPU oracle on the same box:
the GPU factorization (native driver) and oracle/port.py (the reference's
numpy algorithm) on the same A bytes and seed.  Reports identical pivots,
||R - R_oracle|| / ||R_oracle||, the residual of the GPU factorization on a
column sample, and the counters.
Usage: python tools/full_parity.py cfg2 out.json"""
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
cfg = bench.CONFIGS[name]
dev = torch.device("cuda", 0)
A_d = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
A = A_d.cpu().numpy()
A = np.asfortranarray(A)
conf = P.RandomizedConfig(block=cfg["block"], padding=cfg["padding"], seed=0)
t = time.perf_counter()
f = P.rqrcp(A_d, cfg["k"], conf)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t
t = time.perf_counter()
o = port.rqrcp(A, cfg["k"], cfg["block"], cfg["padding"], 0)
t_cpu = time.perf_counter() - t
pf = f.perm.forward.cpu().numpy() if torch.is_tensor(f.perm.forward) else np.asarray(f.perm.forward)
same = pf == o.perm.forward
first_diff = int(np.argmin(same)) if not same.all() else -1
R = f.R.cpu().numpy() if torch.is_tensor(f.R) else np.asarray(f.R)
rerr = float(np.linalg.norm(R - o.R) / np.linalg.norm(o.R))
# residual ||A P - Q R|| on 64 sampled columns (dense Q is not formed)
g = np.random.default_rng(1)
cols = np.sort(g.choice(cfg["n"], 64, replace=False))
E = P.q_columns(f.reflectors.Y, f.reflectors.tau, cfg["m"])
res = float(np.linalg.norm(A[:, pf[cols]] - (E.cpu().numpy() if torch.is_tensor(E) else E) @ R[:, cols])
            / np.linalg.norm(A[:, pf[cols]]))
c = f.counters
out = {"config": name, "m": cfg["m"], "n": cfg["n"], "rank_gpu": int(f.rank), "rank_oracle": int(o.rank),
       "pivots_identical": bool(same.all()), "first_pivot_difference": first_diff,
       "pivot_mismatches": int((~same).sum()), "R_rel_err": rerr, "residual_64_cols": res,
       "counters_gpu": [int(c.gemm_flops), int(c.level2_flops), int(c.resamples)],
       "counters_oracle": [int(o.counters.gemm_flops), int(o.counters.level2_flops),
                           int(o.counters.resamples)],
       "gpu_s": round(t_gpu, 3), "oracle_s": round(t_cpu, 1),
       "note": "same A bytes (generated on the device, copied to the host) and seed; oracle = "
               "oracle/port.py on this box's host cores"}
print(json.dumps(out))
json.dump(out, open(sys.argv[2], "w"), indent=1)
