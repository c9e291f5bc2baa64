"""One fast-panel call (8192 x 64) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
mm, bw = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (8192, 64)
if len(sys.argv) > 3:
    from paper_1509_06820_b200 import _abi
    _abi.load_library().rq_set_option(_abi.handle(0), b"fast_panel_max_ctas", int(sys.argv[3]))
P0 = np.random.default_rng(1).standard_normal((mm, bw))
for _ in range(2):
    P = to_device_fortran(P0, dev); K.panel_qr(P, with_t=False); torch.cuda.synchronize()
print("ok")
