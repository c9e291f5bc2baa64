"""Select v4 vs v5 (register-resident) per-call time and bitwise agreement."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 1)
for ell, b in ((72, 64), (40, 32)):
    for nt in (8192, 4096, 2048, 1024, 512, 128):
        B = to_device_fortran(g.standard_normal((ell, nt)) * np.logspace(0, -3, nt)[None, :], dev)
        r = {"ell": ell, "nt": nt}
        outs = {}
        for v in (0, 1):
            lib.rq_set_option(h, b"select_reg", v)
            r["v5" if v else "v4"] = timeit(lambda: K.select_pivots(B, b))
            o = K.select_pivots(B, b)
            torch.cuda.synchronize()
            outs[v] = [t.cpu().numpy() if torch.is_tensor(t) else t for t in (o if isinstance(o, tuple) else (o,))]
        r["same"] = all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(outs[0], outs[1]))
        print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"select_reg", 1)
