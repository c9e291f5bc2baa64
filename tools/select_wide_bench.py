"""Pivot-selection time on wide samples with few CTAs (cfg5's select beside
the trailing update: ell = 136, nt up to 32768, 44-60 CTAs), shared-memory
kernel (v4) vs the register kernel where it applies.
Usage: python tools/select_wide_bench.py [out.jsonl]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1509_06820_b200 import _abi  # noqa: E402
from paper_1509_06820_b200 import primitives as K  # noqa: E402
from paper_1509_06820_b200.device import to_device_fortran  # noqa: E402

dev = torch.device("cuda", 0)
lib, h = _abi.load_library(), _abi.handle(0)
g = np.random.default_rng(0)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


rows = []
for ell, want in ((136, 128), (72, 64)):
    for nt in (32768, 24576, 16384, 8192, 4096):
        B = to_device_fortran(g.standard_normal((ell, nt)), dev)
        for ctas in (44, 60, 80):
            r = {"ell": ell, "nt": nt, "want": want, "ctas": ctas}
            lib.rq_set_option(h, b"force_select", 1)
            lib.rq_set_option(h, b"select_max_ctas", ctas)
            for reg in (0, 1):
                lib.rq_set_option(h, b"select_reg", reg)
                us = timeit(lambda: K.select_pivots(B, want))
                r["reg_us" if reg else "smem_us"] = round(us, 1)
                r[("reg" if reg else "smem") + "_us_per_step"] = round(us / want, 2)
            rows.append(r)
            print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"force_select", 0)
lib.rq_set_option(h, b"select_max_ctas", 0)
lib.rq_set_option(h, b"select_reg", 1)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")
