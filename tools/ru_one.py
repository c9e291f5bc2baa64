"""One rank-64 update C -= Y X (8192 x 8128, K = 64) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_06820_b200 import primitives as K
dev = torch.device("cuda", 0)
m, n, k = 8192, 8128, 64
C = torch.randn(n, m, dtype=torch.float64, device=dev).t()
Y = torch.randn(k, m, dtype=torch.float64, device=dev).t()
X = torch.randn(n, k, dtype=torch.float64, device=dev).t()
for _ in range(3):
    K.gemm(Y, X, C, alpha=-1.0, beta=1.0)
torch.cuda.synchronize()
print("ok")
