"""Where a cfg3 / cfg4 step spends its time before the first kernel: wall
clock around the pieces of run_native (device copy of A, output allocation,
the host Omega draw) and the whole call.  Usage: python tools/host_breakdown.py cfg3"""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1509_06820_b200 as P
from paper_1509_06820_b200 import _abi, rng as R
from paper_1509_06820_b200.device import to_device_fortran, fmat

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = bench.CONFIGS[name]
dev = torch.device("cuda", 0)
A = bench.device_matrix(cfg["kind"], cfg["m"], cfg["n"], dev, seed=0)
for _ in range(2):
    bench.run_ours(P, cfg, A, None); torch.cuda.synchronize()
def wall(f, n=3):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return round(min(ts), 3)
m, n, k = cfg["m"], cfg["n"], cfg["k"] or min(cfg["m"], cfg["n"])
ell = cfg["block"] + cfg["padding"]
out = {"config": name}
out["whole_call_ms"] = wall(lambda: bench.run_ours(P, cfg, A, None))
out["copy_A_ms"] = wall(lambda: to_device_fortran(A, dev))
out["alloc_outputs_ms"] = wall(lambda: (fmat(m, k, dev), fmat(n, k, dev), fmat(k, n, dev),
                                        torch.empty(n, dtype=torch.int64, device=dev)))
lib = _abi.load_library()
buf = np.empty(ell * m); end = C.c_uint64()
out["omega_draw_ms"] = wall(lambda: lib.rq_omega_fill(0, 0, 0, buf.ctypes.data, ell * m, R.THREADS, C.byref(end)))
out["omega_threads"] = R.THREADS
print(json.dumps(out))
