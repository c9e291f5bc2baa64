import sys, os, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
for force, mm in ((2, 256), (2, 2048), (1, 4096), (1, 8192)):
    lib.rq_set_option(h, b"force_panel", force)
    P0 = to_device_fortran(g.standard_normal((mm, 64)), dev)
    K.panel_qr(P0.clone(), with_t=False)
    lib.rq_set_option(h, b"debug_timers", 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    P = P0.clone()
    e0.record(); K.panel_qr(P, with_t=False); e1.record(); torch.cuda.synchronize()
    buf = (C.c_int64 * 8)()
    lib.rq_debug_read(h, buf, 8)
    lib.rq_set_option(h, b"debug_timers", 0)
    print(json.dumps({"force": force, "mm": mm, "call_us": round(e0.elapsed_time(e1) * 1e3, 1),
                      "cycles_per_step": [round(buf[k] / 64) for k in range(6)],
                      "phases": ["xsync", "reduceQ", "scalars+v", "rowpass", "finish", "loop"]}))
