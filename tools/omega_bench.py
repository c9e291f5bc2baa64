"""Host Omega generation: numpy vs rq_omega_fill at several thread counts."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1509_06820_b200 import _abi
lib = _abi.load_library()
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
n = 72 * 8192
out = np.empty(n); end = C.c_uint64()
g = np.random.Generator(np.random.Philox(key=0))
ts = []
for _ in range(3):
    t = time.perf_counter(); g.standard_normal(n); ts.append(time.perf_counter() - t)
print("numpy %.2f ms" % (min(ts) * 1e3))
for T in (1, 2, 4, 8, 16, 32, 64):
    ts = []
    for _ in range(5):
        t = time.perf_counter(); lib.rq_omega_fill(0, 0, 0, out.ctypes.data, n, T, C.byref(end)); ts.append(time.perf_counter() - t)
    print(T, "%.2f ms" % (min(ts) * 1e3))
print("exact", np.array_equal(out, np.random.Generator(np.random.Philox(key=0)).standard_normal(n)))
