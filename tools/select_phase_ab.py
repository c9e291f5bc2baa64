"""In-kernel phase timers (CTA 0, thread 0) of select v4 vs v5."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
for force, nt in ((2, 256), (2, 1024), (1, 2048), (1, 4096), (1, 8192)):
    lib.rq_set_option(h, b"force_select", force)
    B = to_device_fortran(g.standard_normal((72, nt)), dev)
    for v in (0, 1):
        lib.rq_set_option(h, b"select_reg", v)
        K.select_pivots(B, 64)
        lib.rq_set_option(h, b"debug_timers", 1)
        K.select_pivots(B, 64); torch.cuda.synchronize()
        buf = (C.c_int64 * 8)()
        lib.rq_debug_read(h, buf, 8)
        lib.rq_set_option(h, b"debug_timers", 0)
        n = 5 if v == 0 else 4
        print(json.dumps({"v": "v5" if v else "v4", "force": force, "nt": nt,
                          "cycles_per_step": [round(buf[k] / 64) for k in range(n)],
                          "step_total": round(sum(buf[:n]) / 64)}), flush=True)
lib.rq_set_option(h, b"force_select", 0); lib.rq_set_option(h, b"select_reg", 1)
