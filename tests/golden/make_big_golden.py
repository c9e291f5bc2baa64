"""Golden fixtures at the BASELINE sizes, produced by running the REFERENCE
(/root/reference, build container only) on the exact SURVEY.md §8(d) inputs:

    python tests/golden/make_big_golden.py [cfg2 cfg3 cfg4 cfg5]

Writes tests/golden/big_<cfg>.npz: the sha256 of A's bytes (so the GPU test
knows whether the box rebuilt the same matrix), the reference's permutation,
swap log, counters, resample count, rank, R diagonal and leading rows, and
per config: cfg3's truncation error ||A P - Q_k R_k||_F / ||A||_F, cfg4's
singular value estimates and ||A - U X V^T||_F / ||A||_F.  cfg5 (full RQRCP
takes about an hour on the CPU) stores the reference's TRQRCP with k = 256,
whose pivots equal the first 256 of full RQRCP (reference property,
tests/test_truncated.py:35-46 upstream)."""

from __future__ import annotations

import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import recipes  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main(names):
    import rqrcp as rq
    for name in names:
        t0 = time.perf_counter()
        A = recipes.build(name)
        t_build = time.perf_counter() - t0
        driver, k, block, padding, desc = recipes.CONFIGS[name]
        if name == "cfg5":
            driver, k = "trqrcp", 256
        cfg = rq.RandomizedConfig(block=block, padding=padding, seed=0)
        t0 = time.perf_counter()
        f = getattr(rq, driver)(A, k=k, config=cfg)
        t_ref = time.perf_counter() - t0
        rec = dict(config=name, driver=driver, k=-1 if k is None else k, block=block,
                   padding=padding, seed=0, m=A.shape[0], n=A.shape[1], A_sha=recipes.sha(A),
                   ref_seconds=t_ref, build_seconds=t_build, host_cpu=cpu_model(),
                   threads=os.cpu_count(), rank=f.rank)
        c = f.counters
        rec.update(gemm_flops=c.gemm_flops, level2_flops=c.level2_flops,
                   bytes_touched=c.bytes_touched, resamples=c.resamples)
        nA = np.linalg.norm(A)
        if driver == "tuxv":
            rec["sv"] = f.singular_values()
            rec["approx_err"] = np.linalg.norm(A - f.approx()) / nA
        else:
            rec["perm"] = np.asarray(f.perm.forward, dtype=np.int64)
            rec["swaps"] = np.asarray(f.perm.swaps, dtype=np.int64).reshape(-1, 2)
            rec["R_diag"] = np.diag(f.R).copy()
            rec["R_head"] = f.R[:4].copy()
            rec["R_sha"] = recipes.sha(f.R)
            if driver == "trqrcp":
                Q = f.q_factor()
                rec["trunc_err"] = np.linalg.norm(A[:, f.perm.forward] - Q @ f.R) / nA
        np.savez_compressed(os.path.join(HERE, f"big_{name}.npz"), **rec)
        print(name, driver, f"A sha {rec['A_sha'][:12]} build {t_build:.1f}s ref {t_ref:.1f}s",
              {k_: rec[k_] for k_ in ("rank", "resamples", "trunc_err", "approx_err") if k_ in rec},
              flush=True)
        del A, f


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"])
