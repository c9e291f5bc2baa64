"""Phase / serial-section timers (cycles, CTA 0) of the LAST fast panel of a
truncated-count RQRCP run, i.e. the panel as the driver configures it (T, the
sample update's M and block_finish's A1/A2 on, CTA cap from panel_split)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_06820_b200 as P
from paper_1509_06820_b200 import _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
n = 8192
A = to_device_fortran(np.random.default_rng(0).standard_normal((n, n)), dev)
cfg = P.RandomizedConfig(block=64, padding=8, seed=0)
names = ["gramA", "reduce1", "chol+inv", "gramB", "reduce2", "serial2_lu", "serial2_m", "applyC"]
for k in (64, 2048 + 64, 4096 + 64, 6144 + 64, 7168 + 64):
    lib.rq_set_option(h, b"debug_timers", 1)
    for _ in range(2):
        f = P.rqrcp(A, k, cfg); torch.cuda.synchronize()
    buf = (C.c_int64 * 64)()
    lib.rq_debug_read(h, buf, 64)
    print(json.dumps({"mm": n - k + 64, "cycles": dict(zip(names, list(buf)[8:16])), "total": sum(list(buf)[8:16]),
                      "sub": list(buf)[16:26]}), flush=True)
    lib.rq_set_option(h, b"debug_timers", 0)
