"""GPU qr_blocked (this library: panel kernels + tc_gemm block reflections,
csrc/driver.cu qr_blocked) against cuSOLVER dgeqrf on the same device matrix
-- the paper's "performance limit" comparator for unpivoted blocked QR
(SURVEY §8(f)3).  cuSOLVER is the yardstick here, never on the product path.
Times with CUDA events after warm-up; reports GFLOP/s of the standard
Householder count 2mn^2 - 2n^3/3 and the residual of our factorization.

    python tools/qr_vs_cusolver.py out.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_06820_b200 as P  # noqa: E402
from paper_1509_06820_b200.device import fmat  # noqa: E402

SHAPES = [(8192, 8192, 64), (8192, 8192, 32), (16384, 4096, 64), (20000, 256, 32),
          (12000, 256, 32), (4096, 4096, 64)]


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(out):
    dev = torch.device("cuda", 0)
    torch.backends.cuda.preferred_linalg_library("cusolver")
    rows = []
    g = torch.Generator(device=dev).manual_seed(0)
    for m, n, b in SHAPES:
        A = fmat(m, n, dev)
        A.copy_(torch.randn((n, m), dtype=torch.float64, device=dev, generator=g).t())
        flops = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
        ms_ours = timeit(lambda: P.qr_blocked(A, None, b))
        ms_cus = timeit(lambda: torch.geqrf(A))
        f = P.qr_blocked(A, None, b)
        k = min(m, n)
        Q = f.q_factor()
        res = float(torch.linalg.matrix_norm(A - Q @ f.R) / torch.linalg.matrix_norm(A))
        r = {"m": m, "n": n, "b": b, "ours_ms": round(ms_ours, 3), "cusolver_dgeqrf_ms": round(ms_cus, 3),
             "ours_gflops": round(flops / ms_ours / 1e6, 1),
             "cusolver_gflops": round(flops / ms_cus / 1e6, 1),
             "ratio_ours_over_cusolver": round(ms_cus / ms_ours, 3), "residual": res, "k": k}
        rows.append(r)
        print(json.dumps(r), flush=True)
        del A, f, Q
        torch.cuda.empty_cache()
    with open(out, "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/qr_vs_cusolver.jsonl")
