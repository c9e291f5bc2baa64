"""Sample-update kernel time vs width (CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
g = np.random.default_rng(0)
for nt in (8128, 4096, 1024, 256):
    ell, b = 72, 64
    S = to_device_fortran(g.standard_normal((ell, nt + b)), dev)
    R11 = to_device_fortran(np.triu(g.standard_normal((b, b))) + 8 * np.eye(b), dev)
    R12 = to_device_fortran(g.standard_normal((b, nt)), dev)
    K.sample_update(S, b, R11, R12, 1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        K.sample_update(S, b, R11, R12, 1.0)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"nt": nt, "us_per_call_incl_wrapper": round(e0.elapsed_time(e1) / 10 * 1e3, 1)}))
