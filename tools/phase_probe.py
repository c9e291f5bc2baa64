import sys, os, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
for force, nt in ((2, 256), (2, 1024), (1, 4096), (1, 8192)):
    lib.rq_set_option(h, b"force_select", force)
    B = to_device_fortran(g.standard_normal((72, nt)), dev)
    K.select_pivots(B, 64)
    lib.rq_set_option(h, b"debug_timers", 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); K.select_pivots(B, 64); e1.record(); torch.cuda.synchronize()
    buf = (C.c_int64 * 8)()
    lib.rq_debug_read(h, buf, 8)
    lib.rq_set_option(h, b"debug_timers", 0)
    tot = sum(buf[:5])
    print(json.dumps({"force": force, "nt": nt, "call_us": e0.elapsed_time(e1) * 1e3,
                      "cycles_per_step": [round(buf[k] / 64) for k in range(5)], "total_cycles": tot,
                      "phases": ["winner", "reflector", "apply", "publish", "xsync"]}))
