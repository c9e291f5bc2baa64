"""One select call for ncu: python tools/select_one.py nt force(1 grid / 2 cluster) [max_ctas] [ell] [want] [select_reg]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
lib = _abi.load_library(); h = _abi.handle(0)
nt, force = int(sys.argv[1]), int(sys.argv[2])
lib.rq_set_option(h, b"force_select", force)
if len(sys.argv) > 3:
    lib.rq_set_option(h, b"select_max_ctas", int(sys.argv[3]))
ell = int(sys.argv[4]) if len(sys.argv) > 4 else 72
want = int(sys.argv[5]) if len(sys.argv) > 5 else 64
if len(sys.argv) > 6:
    lib.rq_set_option(h, b"select_reg", int(sys.argv[6]))
B = to_device_fortran(np.random.default_rng(0).standard_normal((ell, nt)), torch.device("cuda", 0))
for _ in range(2):
    K.select_pivots(B, want)
torch.cuda.synchronize()
print("ok")
