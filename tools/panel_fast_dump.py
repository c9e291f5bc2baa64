"""Dump fast-panel outputs (R, Y, tau, T) for a fixed set of panels, plus one
full RQRCP, to an npz; `--compare old.npz` checks a rebuilt library against
it bit for bit.  Usage: python tools/panel_fast_dump.py out.npz [--compare ref.npz]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1509_06820_b200 as PK
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import to_device_fortran

dev = torch.device("cuda", 0)
out = {}
for mm, bw, seed in ((8192, 64, 1), (4096, 64, 2), (1000, 61, 3), (777, 32, 4), (300, 16, 5),
                     (150, 13, 6), (5000, 48, 7), (2048, 57, 8), (96, 8, 9)):
    g = np.random.default_rng(seed)
    A = g.standard_normal((mm, bw)) * np.exp(g.uniform(-2, 2, bw))
    P = to_device_fortran(A, dev)
    Y, tau, T, usable, l2 = K.panel_qr(P, with_t=True)
    key = f"{mm}_{bw}"
    out[key + "_R"] = P.cpu().numpy()
    out[key + "_Y"] = Y.cpu().numpy()
    out[key + "_tau"] = tau.cpu().numpy()
    out[key + "_T"] = T.cpu().numpy()
A = np.random.default_rng(11).standard_normal((1500, 1300))
f = PK.rqrcp(A, None, PK.RandomizedConfig(block=64, padding=8, seed=0))
out["rq_R"] = f.R
out["rq_perm"] = np.asarray(f.perm.forward)
np.savez(sys.argv[1], **out)
if "--compare" in sys.argv:
    ref = np.load(sys.argv[sys.argv.index("--compare") + 1])
    bad = [k for k in ref.files if not np.array_equal(ref[k], out[k])]
    print("bitwise identical" if not bad else f"DIFFER: {bad}")
    for k in bad:
        print(k, float(np.max(np.abs(ref[k] - out[k]))))
