"""Grid v5 select exchange knobs: per-step cycles for key stride x poll back-off."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
for nt, ctas in ((8128, 56), (8128, 0), (4096, 56), (1024, 56)):
    B = to_device_fortran(g.standard_normal((72, nt)), dev)
    lib.rq_set_option(h, b"force_select", 1)
    lib.rq_set_option(h, b"select_max_ctas", ctas)
    for ks in (1, 16):
        for ns in (0, 32, 100):
            lib.rq_set_option(h, b"sel_kstride", ks); lib.rq_set_option(h, b"sel_poll_ns", ns)
            lib.rq_set_option(h, b"debug_timers", 1)
            for _ in range(3):
                K.select_pivots(B, 64)
            torch.cuda.synchronize()
            buf = (C.c_int64 * 64)()
            lib.rq_debug_read(h, buf, 64)
            steps = max(buf[7], 1)
            lib.rq_set_option(h, b"debug_timers", 0)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(5):
                K.select_pivots(B, 64)
            ev[1].record(); torch.cuda.synchronize()
            print(json.dumps({"nt": nt, "ctas": ctas, "kstride": ks, "poll_ns": ns,
                              "per_step": [round(buf[k] / steps) for k in range(4)],
                              "us_per_call": round(ev[0].elapsed_time(ev[1]) / 5 * 1e3, 1)}), flush=True)
lib.rq_set_option(h, b"force_select", 0); lib.rq_set_option(h, b"select_max_ctas", 0)
