"""Time grid vs cluster variants of select and panel across sizes (CUDA events)."""
import sys, os, json
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
    return e0.elapsed_time(e1) / reps * 1e3
out = []
for ell, b in ((72, 64), (40, 32), (136, 128)):
    for nt in (8192, 6144, 4096, 3072, 2048, 1024, 512, 256):
        if nt < b: continue
        B = to_device_fortran(g.standard_normal((ell, nt)), dev)
        r = {"kind": "select", "ell": ell, "nt": nt, "want": b}
        for v, nm in ((1, "grid"), (2, "cluster")):
            lib.rq_set_option(h, b"force_select", v)
            r[nm] = timeit(lambda: K.select_pivots(B, b))
        out.append(r); print(json.dumps(r), flush=True)
for bw in (64, 32, 128):
    for mm in (8192, 6144, 4096, 3072, 2048, 1024, 512, 256):
        if mm < bw: continue
        P0 = g.standard_normal((mm, bw))
        r = {"kind": "panel", "mm": mm, "bw": bw}
        for v, nm in ((1, "grid"), (2, "cluster")):
            lib.rq_set_option(h, b"force_panel", v)
            P = to_device_fortran(P0, dev)
            r[nm] = timeit(lambda: K.panel_qr(P.clone()))
        out.append(r); print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"force_select", 0); lib.rq_set_option(h, b"force_panel", 0)
