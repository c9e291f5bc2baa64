"""Phase timers (cycles, CTA 0) of the fast panel kernel."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import _abi
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
lib.rq_set_option(h, b"debug_timers", 1)
names = ["gramA", "reduce1", "chol+inv", "gramB", "reduce2", "serial2_lu", "serial2_m", "applyC"]
pads = [int(x) for x in os.environ.get("PADS", "1").split(",")]
cases = [(mm, bw, q, pad) for pad in pads for (mm, bw, q) in
         ((8192, 64, 0), (8192, 64, 48), (4096, 64, 48), (2048, 64, 0), (1024, 64, 0), (8192, 32, 48))]
for mm, bw, q, pad in cases:
    lib.rq_set_option(h, b"fast_panel_max_ctas", q)
    lib.rq_set_option(h, b"fast_panel_pad", pad)
    P0 = np.random.default_rng(1).standard_normal((mm, bw))
    for _ in range(3):
        P = to_device_fortran(P0, dev); K.panel_qr(P, with_t=False); torch.cuda.synchronize()
    buf = (C.c_int64 * 64)()
    lib.rq_debug_read(h, buf, 64)
    print(json.dumps({"mm": mm, "bw": bw, "q": q, "pad": pad, "cycles": dict(zip(names, list(buf)[8:16])), "sub": list(buf)[16:26], "chol_steps": list(buf)[28:31]}))
lib.rq_set_option(h, b"debug_timers", 0)
lib.rq_set_option(h, b"fast_panel_pad", 4)
