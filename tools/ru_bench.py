"""Rank-64 update C -= Y X throughput (CUDA events) at a few trailing shapes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_06820_b200 import primitives as K, _abi
dev = torch.device("cuda", 0)
lib, h = _abi.load_library(), _abi.handle(0)
opts = [kv.split("=") for kv in sys.argv[1:]]
for k_, v_ in opts:
    _abi.check(lib.rq_set_option(h, k_.encode(), int(v_)))
out = {"opts": sys.argv[1:]}
for m, n in ((8192, 8128), (6144, 6080), (4096, 4032), (2048, 1984)):
    k = 64
    C = torch.randn(n, m, dtype=torch.float64, device=dev).t()
    Y = torch.randn(k, m, dtype=torch.float64, device=dev).t()
    X = torch.randn(n, k, dtype=torch.float64, device=dev).t()
    for _ in range(3):
        K.gemm(Y, X, C, alpha=-1.0, beta=1.0)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 10
    ev[0].record()
    for _ in range(reps):
        K.gemm(Y, X, C, alpha=-1.0, beta=1.0)
    ev[1].record(); torch.cuda.synchronize()
    us = ev[0].elapsed_time(ev[1]) / reps * 1e3
    out[f"{m}x{n}"] = {"us": round(us, 1), "TF/s": round(2 * m * n * k / us / 1e6, 2),
                       "GB/s": round(16 * m * n / us / 1e3, 0)}
print(json.dumps(out))
