"""Run one select + one panel + one sample update + one update GEMM at cfg2's first-block shapes (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import to_device_fortran, fmat
dev = torch.device("cuda", 0)
g = np.random.default_rng(0)
B = to_device_fortran(g.standard_normal((72, 8192)), dev)
P0 = g.standard_normal((8192, 64))
C = to_device_fortran(g.standard_normal((8192, 8128)), dev)
Y = to_device_fortran(g.standard_normal((8192, 64)), dev)
X = to_device_fortran(g.standard_normal((64, 8128)), dev)
for it in range(2):
    S, piv, got, *_ = K.select_pivots(B, 64)
    P = to_device_fortran(P0, dev)
    K.panel_qr(P)
    K.gemm(Y, X, C, alpha=-1.0, beta=1.0)
    K.gemm(Y, C, fmat(64, 8128, dev), transa=True)
torch.cuda.synchronize()
print("probe ok", got)
