"""One inner GEMM G = Y^T C (64 x 8128, K = 8192) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import fmat
dev = torch.device("cuda", 0)
m, n, k = 8192, 8128, 64
C = torch.randn(n, m, dtype=torch.float64, device=dev).t()
Y = torch.randn(k, m, dtype=torch.float64, device=dev).t()
G = fmat(k, n, dev)
for _ in range(3):
    K.gemm(Y, C, G, transa=True)
torch.cuda.synchronize()
print("ok")
