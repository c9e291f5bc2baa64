import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_06820_b200 import primitives as K, _abi
from paper_1509_06820_b200.device import to_device_fortran
from oracle import port
dev = torch.device("cuda", 0)
lib = _abi.load_library(); h = _abi.handle(0)
for mm, bw in ((256, 64), (300, 32), (1000, 32), (4096, 64), (8192, 64)):
    P0 = np.random.default_rng(mm + bw).standard_normal((mm, bw))
    Pc = np.asfortranarray(P0.copy()); Yo, to = port.panel_qr(Pc)
    for force in (1, 2):
        lib.rq_set_option(h, b"force_panel", force)
        try:
            P = to_device_fortran(P0, dev); Y, tau, T, usable, _ = K.panel_qr(P)
            errR = np.linalg.norm(P.cpu().numpy() - Pc) / np.linalg.norm(P0)
            bad = np.argwhere(np.abs(P.cpu().numpy() - Pc) > 1e-10)
            print(mm, bw, "grid" if force == 1 else "cluster", f"{errR:.2e}", bad[:3].tolist() if len(bad) else "")
        except Exception as e:
            print(mm, bw, force, "EXC", e)
lib.rq_set_option(h, b"force_panel", 0)
