"""Host-path breakdown of one rqrcp(numpy A) call (cfg2): H2D, device
factorization, packaging (D2H + Python)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1509_06820_b200 as P
from paper_1509_06820_b200 import randomized as Rz
from paper_1509_06820_b200.device import to_device_fortran
cfg = bench.CONFIGS["cfg2"]
dev = torch.device("cuda", 0)
A = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
Ah = torch.empty((cfg["n"], cfg["m"]), dtype=torch.float64).pin_memory().t()
Ah.copy_(A)
Ahost = Ah.numpy()
config = P.RandomizedConfig(block=cfg["block"], padding=cfg["padding"], seed=0)
def sync(): torch.cuda.synchronize()
for rep in range(4):
    t0 = time.perf_counter()
    W = to_device_fortran(Ahost, dev); sync(); t1 = time.perf_counter()
    out = Rz.run_native(W, cfg["k"] or min(cfg["m"], cfg["n"]), config, variant=0, ell=cfg["block"] + cfg["padding"], width=cfg["block"]); sync(); t2 = time.perf_counter()
    pk = Rz.package(out, True, True); t3 = time.perf_counter()
    f = P.rqrcp(Ahost, cfg["k"], config); t4 = time.perf_counter()
    print(f"rep {rep}: h2d {1e3*(t1-t0):.1f} ms  factor {1e3*(t2-t1):.1f} ms  package {1e3*(t3-t2):.1f} ms  | full rqrcp(numpy) {1e3*(t4-t3):.1f} ms", flush=True)
