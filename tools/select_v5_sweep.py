"""v5 select: cluster vs grid per-call kernel time (in-kernel phase timers off) vs nt."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
lib.rq_set_option(h, b"profile_trace", 0)
g = np.random.default_rng(0)
import ctypes as C
def ktime(fn, reps=5):
    fn(); torch.cuda.synchronize()
    lib.rq_profile_reset(h); lib.rq_profile_enable(h, 1)
    for _ in range(reps): fn()
    torch.cuda.synchronize(); lib.rq_profile_enable(h, 0)
    L = (C.c_int64 * 9)(); MS = (C.c_double * 9)()
    lib.rq_profile_read(h, L, MS, None, None)
    i = _abi.PROF_NAMES.index("select")
    return round(MS[i] / max(L[i], 1) * 1e3, 1)
for nt in (768, 1024, 1280, 1536, 2048, 3072):
    B = to_device_fortran(g.standard_normal((72, nt)), dev)
    r = {"nt": nt}
    for v, nm in ((1, "grid148"), (2, "cluster16")):
        lib.rq_set_option(h, b"force_select", v)
        r[nm] = ktime(lambda: K.select_pivots(B, 64))
    lib.rq_set_option(h, b"force_select", 1); lib.rq_set_option(h, b"select_max_ctas", 56)
    r["grid56"] = ktime(lambda: K.select_pivots(B, 64))
    lib.rq_set_option(h, b"select_max_ctas", 0)
    print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"force_select", 0)
