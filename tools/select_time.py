"""Per-call select kernel time (CUDA events) for a few widths / CTA caps.
RQ_LIB_PATH selects the library build (A/B of two builds)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
out = {}
for nt, ctas in ((8128, 56), (7000, 56), (8128, 0), (4096, 56), (2048, 56), (1024, 56), (1024, 0)):
    B = to_device_fortran(g.standard_normal((72, nt)), dev)
    lib.rq_set_option(h, b"force_select", 1 if ctas or nt > 1024 else 0)
    lib.rq_set_option(h, b"select_max_ctas", ctas)
    for _ in range(3):
        K.select_pivots(B, 64)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(10):
        K.select_pivots(B, 64)
    ev[1].record(); torch.cuda.synchronize()
    out[f"{nt}@{ctas}"] = round(ev[0].elapsed_time(ev[1]) / 10 * 1e3, 1)
print(json.dumps({"lib": os.environ.get("RQ_LIB_PATH", "new"), "us": out}))
lib.rq_set_option(h, b"force_select", 0); lib.rq_set_option(h, b"select_max_ctas", 0)
