"""Per-step phase cycles of the v5 select (CTA 0 thread 0 timers):
[winner+reflector, apply+downdate, block key+publish, exchange].
Usage: python tools/select_phases.py"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
g = np.random.default_rng(0)
for ll in [int(x) for x in os.environ.get("FUSED", "1").split(",")]:
  lib.rq_set_option(h, b"select_fused", ll)
  for nt, force, ctas in ((8128, 1, 44), (6000, 1, 44), (4096, 1, 80), (2048, 1, 80), (2048, 2, 0), (1024, 2, 0), (512, 2, 0), (256, 2, 0), (1024, 1, 80), (512, 1, 80)):
      B = to_device_fortran(g.standard_normal((72, nt)), dev)
      lib.rq_set_option(h, b"force_select", force)
      lib.rq_set_option(h, b"select_max_ctas", ctas)
      lib.rq_set_option(h, b"debug_timers", 1)
      for _ in range(3):
          K.select_pivots(B, 64)
      torch.cuda.synchronize()
      buf = (C.c_int64 * 64)()
      lib.rq_debug_read(h, buf, 64)
      steps = max(buf[7], 1)
      print(json.dumps({"fused": ll, "nt": nt, "force": force, "ctas": ctas, "winner_split": [round(buf[32 + k] / steps) for k in range(4)],
                        "per_step": [round(buf[k] / steps) for k in range(4)],
                        "total_per_step": round(sum(buf[k] for k in range(4)) / steps)}), flush=True)
      lib.rq_set_option(h, b"debug_timers", 0)
lib.rq_set_option(h, b"force_select", 0); lib.rq_set_option(h, b"select_max_ctas", 0)
