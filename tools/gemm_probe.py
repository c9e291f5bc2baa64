"""Time the rank-64 update (persistent vs generic) and the inner GEMM at cfg2 block-0 shapes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import fmat
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for (m, n, k) in ((8192, 8128, 64), (4096, 4032, 64), (2048, 1984, 64), (16384, 16256, 64), (8192, 8064, 32)):
    C = torch.randn(n, m, dtype=torch.float64, device=dev).t()
    Y = torch.randn(k, m, dtype=torch.float64, device=dev).t()
    X = torch.randn(n, k, dtype=torch.float64, device=dev).t()
    ref = C - Y @ X
    r = {"m": m, "n": n, "k": k}
    for flag in (1, 0):
        lib.rq_set_option(h, b"use_rank_update", flag)
        Cw = C.clone()
        K.gemm(Y, X, Cw, alpha=-1.0, beta=1.0)
        r[f"err_{flag}"] = float((Cw - ref).abs().max())
        us = timeit(lambda: K.gemm(Y, X, Cw, alpha=-1.0, beta=1.0))
        r[f"us_{'persist' if flag else 'generic'}"] = round(us, 1)
        r[f"tflops_{'persist' if flag else 'generic'}"] = round(2 * m * n * k / us / 1e6, 2)
    G = fmat(k, n, dev)
    us = timeit(lambda: K.gemm(Y, C, G, transa=True))
    r["inner_us"] = round(us, 1); r["inner_tflops"] = round(2 * m * n * k / us / 1e6, 2)
    print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"use_rank_update", 1)
