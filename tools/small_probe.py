import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
lib.rq_set_option(h, b"force_select", 2); lib.rq_set_option(h, b"force_panel", 2)
g = np.random.default_rng(0)
B = to_device_fortran(g.standard_normal((72, 256)), dev)
P = to_device_fortran(g.standard_normal((256, 64)), dev)
for _ in range(2):
    K.select_pivots(B, 64)
    K.panel_qr(P.clone())
torch.cuda.synchronize(); print("ok")
