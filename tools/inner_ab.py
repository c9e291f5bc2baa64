import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import fmat
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for (m, n, k) in ((8192, 8128, 64), (4096, 4032, 64), (16384, 16256, 64), (8192, 8192, 72)):
    C = torch.randn(n, m, dtype=torch.float64, device=dev).t()
    Y = torch.randn(k, m, dtype=torch.float64, device=dev).t()
    G = fmat(k, n, dev)
    r = {"m": m, "n": n, "k": k}
    for v in (0, 1):
        lib.rq_set_option(h, b"gemm_vec16", v)
        us = timeit(lambda: K.gemm(Y, C, G, transa=True))
        r[f"inner_vec{v}"] = round(2 * m * n * k / us / 1e6, 2)
    Om = torch.randn(m, k, dtype=torch.float64, device=dev).t()   # sketch: Omega (k x m) N
    B = fmat(k, n, dev)
    for v in (0, 1):
        lib.rq_set_option(h, b"gemm_vec16", v)
        us = timeit(lambda: K.gemm(Om, C, B))
        r[f"sketch_vec{v}"] = round(2 * m * n * k / us / 1e6, 2)
    print(json.dumps(r), flush=True)
lib.rq_set_option(h, b"gemm_vec16", 1)
