"""Select time vs CTA cap of the grid variant (CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 1)
lib.rq_set_option(h, b"force_select", 1)
for nt in (8192, 6144, 4096, 2048, 1024):
    B = to_device_fortran(g.standard_normal((72, nt)), dev)
    r = {"nt": nt}
    for cap in (148, 112, 96, 64, 48, 32, 16):
        lib.rq_set_option(h, b"select_max_ctas", cap)
        r[cap] = timeit(lambda: K.select_pivots(B, 64))
    lib.rq_set_option(h, b"force_select", 2); r["cluster"] = timeit(lambda: K.select_pivots(B, 64))
    lib.rq_set_option(h, b"force_select", 1)
    print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"select_max_ctas", 0); lib.rq_set_option(h, b"force_select", 0)
