"""tc_gemm (csrc/tc_gemm.cu) against cuBLAS (torch.matmul) on the hot path's
product shapes: accuracy and TFLOP/s per tile family.

    python tools/tc_bench.py [--quick] [--variants 0,1,2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1509_06820_b200 import _abi  # noqa: E402
from paper_1509_06820_b200 import primitives as K  # noqa: E402

SHAPES = [
    # name, ta, tb, M, N, K, alpha, beta
    ("sketch_cfg2", 0, 0, 72, 8192, 8192, 1.0, 0.0),
    ("sketch_cfg3", 0, 0, 72, 16384, 16384, 1.0, 0.0),
    ("sketch_cfg5", 0, 0, 136, 32768, 32768, 1.0, 0.0),
    ("sketch_cfg1", 0, 0, 40, 1000, 1000, 1.0, 0.0),
    ("inner_b128_cfg5", 1, 0, 128, 32640, 32768, 1.0, 0.0),
    ("inner_b128_mid", 1, 0, 128, 16256, 16384, 1.0, 0.0),
    ("inner_b64_cfg2", 1, 0, 64, 8128, 8192, 1.0, 0.0),
    ("trq_G_cfg3", 1, 0, 64, 16320, 16384, 1.0, 0.0),
    ("tuxv_AV", 0, 0, 20000, 256, 12000, 1.0, 0.0),
    ("tuxv_UtA", 1, 0, 256, 12000, 20000, 1.0, 0.0),
    ("square_8192", 0, 0, 8192, 8192, 8192, 1.0, 0.0),
    ("trq_ZWt", 0, 1, 72, 16384, 512, -1.0, 1.0),
    ("trq_YWt", 0, 1, 16384, 64, 512, -1.0, 1.0),
    ("qrb_update", 0, 0, 12000, 224, 32, -1.0, 1.0),
    ("qrb_X", 1, 0, 32, 224, 32, 1.0, 0.0),
    ("ru_b64_cfg2", 0, 0, 8128, 8128, 64, -1.0, 1.0),
    ("ru_b64_half", 0, 0, 4032, 4032, 64, -1.0, 1.0),
    ("ru_b128_mid", 0, 0, 16256, 16256, 128, -1.0, 1.0),
]


def fmat_from(buf, rows, cols):
    need = rows * cols
    return buf[:need].view(cols, rows).t()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--variants", default="")
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _abi.load_library()
    h = _abi.handle(0)
    big = torch.randn(32768 * 32768 + (1 << 20), dtype=torch.float64, device=dev) if not a.quick else None
    variants = [int(v) for v in a.variants.split(",") if v != ""]

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    for name, ta, tb, M, N, Kd, alpha, beta in SHAPES:
        if a.only and name not in a.only.split(","):
            continue
        if a.quick and M * N + M * Kd + Kd * N > 3e8:
            continue
        ar, ac = (Kd, M) if ta else (M, Kd)
        br, bc = (N, Kd) if tb else (Kd, N)
        if big is not None and ar * ac > 4e8:
            A = fmat_from(big, ar, ac)
        else:
            A = torch.randn(ac, ar, dtype=torch.float64, device=dev).t()
        if big is not None and br * bc > 4e8:
            B = fmat_from(big, br, bc)
        else:
            B = torch.randn(bc, br, dtype=torch.float64, device=dev).t()
        C0 = torch.randn(N, M, dtype=torch.float64, device=dev).t()
        opA = A.t() if ta else A
        opB = B.t() if tb else B
        ref = alpha * (opA @ opB) + beta * C0 if beta != 0 else alpha * (opA @ opB)
        flops = 2.0 * M * N * Kd
        r = {"shape": name, "M": M, "N": N, "K": Kd, "ta": ta, "tb": tb}
        Cb = C0.clone()

        def cub():
            torch.addmm(Cb, opA, opB, beta=beta, alpha=alpha, out=Cb) if beta != 0 else \
                torch.mm(opA, opB, out=Cb)
        us = timeit(cub, a.reps)
        r["cublas_tf"] = round(flops / us / 1e6, 2)
        scale = float(ref.abs().max())
        for label, opts in [("auto", {"tc_variant": -1})] + \
                [(f"v{v}", {"tc_variant": v}) for v in variants] + [("cpasync", {"tc_tma": 0}), ("rubig", {"ru_tma": 0}), ("ru2", {"ru_tma": 2}), ("ru3", {"ru_tma": 3}), ("old", {"use_tc": 0}),
                                                                     ("noru", {"use_rank_update": 0})]:
            for k_, v_ in opts.items():
                _abi.check(lib.rq_set_option(h, k_.encode(), v_))
            C = C0.clone()
            K.gemm(A, B, C, alpha=alpha, beta=beta, transa=bool(ta), transb=bool(tb))
            torch.cuda.synchronize()
            err = float((C - ref).abs().max()) / scale
            us = timeit(lambda: K.gemm(A, B, C, alpha=alpha, beta=beta, transa=bool(ta),
                                       transb=bool(tb)), a.reps)
            r[f"{label}_tf"] = round(flops / us / 1e6, 2)
            r[f"{label}_err"] = float(f"{err:.2e}")
            _abi.check(lib.rq_set_option(h, b"use_tc", 1))
            _abi.check(lib.rq_set_option(h, b"use_rank_update", 1))
            _abi.check(lib.rq_set_option(h, b"tc_tma", 1))
            _abi.check(lib.rq_set_option(h, b"ru_tma", 2))
            _abi.check(lib.rq_set_option(h, b"tc_variant", -1))
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
