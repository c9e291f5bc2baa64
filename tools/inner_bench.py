"""H = P^T C (64 x N, K rows) throughput: stream-K kernel vs the generic GEMM."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_06820_b200 import primitives as K_, _abi
dev = torch.device("cuda", 0)
lib, h = _abi.load_library(), _abi.handle(0)
for v in (0, 1):
    _abi.check(lib.rq_set_option(h, b"inner_kernel", v))
    out = {"inner_kernel": v}
    for k, n in ((8128, 8128), (6080, 6080), (4032, 4032), (1984, 1984), (960, 960)):
        P = torch.randn(64, k, dtype=torch.float64, device=dev).t()
        C = torch.randn(n, k, dtype=torch.float64, device=dev).t()
        H = torch.zeros(n, 64, dtype=torch.float64, device=dev).t()
        for _ in range(3):
            K_.gemm(P, C, H, transa=True)
        ref = (P.t() @ C)
        err = float((H - ref).abs().max() / ref.abs().max())
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(10):
            K_.gemm(P, C, H, transa=True)
        ev[1].record(); torch.cuda.synchronize()
        us = ev[0].elapsed_time(ev[1]) / 10 * 1e3
        out[f"{k}x{n}"] = {"us": round(us, 1), "TF/s": round(2 * 64 * n * k / us / 1e6, 2), "err": err}
    print(json.dumps(out))
_abi.check(lib.rq_set_option(h, b"inner_kernel", 1))
