"""Exact (column-by-column) panel kernel time vs rows per CTA of the cluster
variant, and the T factor's time.  Usage: python tools/panel_rows_sweep.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import _abi
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
lib.rq_set_option(h, b"fast_panel", 0)


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 1)


for mm in (128, 256, 512, 1024, 2048, 3072):
    P0 = to_device_fortran(np.random.default_rng(mm).standard_normal((mm, 64)), dev)
    r = {"mm": mm}
    for rpc in (128, 256, 512, 1024):
        lib.rq_set_option(h, b"panel_rows_per_cta", rpc)
        r[rpc] = timeit(lambda: K.panel_qr(P0.clone(), with_t=False))
        if rpc == 128:
            r["with_T"] = timeit(lambda: K.panel_qr(P0.clone(), with_t=True))
    r["clone"] = timeit(lambda: P0.clone())
    print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"panel_rows_per_cta", 128)
lib.rq_set_option(h, b"fast_panel", 1)
