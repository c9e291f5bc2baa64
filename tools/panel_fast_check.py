"""Fast (CholeskyQR2 + reconstruction) vs exact panel: errors against the
oracle and per-call time.  Usage: python tools/panel_fast_check.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import port
from paper_1509_06820_b200 import _abi
from paper_1509_06820_b200 import primitives as K
from paper_1509_06820_b200.device import to_device_fortran

dev = torch.device("cuda", 0)
lib = _abi.load_library()
h = _abi.handle(0)


def case(kind, mm, bw, seed):
    g = np.random.default_rng(seed)
    P = g.standard_normal((mm, bw))
    if kind == "dup":
        P[:, bw // 2] = P[:, 1]
    elif kind == "scaled":
        P[:, -1] *= 1e-9
    elif kind == "zero":
        P[:, 3] = 0.0
    elif kind == "graded":
        P *= np.logspace(0, -2, bw)[None, :]
    return P


def run(P0, fast):
    lib.rq_set_option(h, b"fast_panel", fast)
    P = to_device_fortran(P0, dev)
    Y, tau, T, usable, l2 = K.panel_qr(P)
    torch.cuda.synchronize()
    return P.cpu().numpy(), Y.cpu().numpy(), tau.cpu().numpy(), T.cpu().numpy(), usable, l2


def timed(P0, fast, reps=20):
    lib.rq_set_option(h, b"fast_panel", fast)
    P = to_device_fortran(P0, dev)
    work = P.clone()
    for _ in range(3):
        work.copy_(P)
        K.panel_qr(work)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    tot = 0.0
    for _ in range(reps):
        work.copy_(P)
        ev[0].record()
        K.panel_qr(work)
        ev[1].record()
        torch.cuda.synchronize()
        tot += ev[0].elapsed_time(ev[1])
    return tot / reps * 1e3


for kind, mm, bw in [("gauss", 8192, 64), ("gauss", 4096, 64), ("gauss", 1000, 32),
                     ("gauss", 257, 17), ("gauss", 130, 64), ("graded", 8192, 64),
                     ("dup", 2048, 64), ("scaled", 2048, 64), ("zero", 2048, 32),
                     ("gauss", 32768, 64), ("gauss", 16384, 32)]:
    P0 = case(kind, mm, bw, mm + bw)
    Pc = np.asfortranarray(P0.copy())
    Yo, to = port.panel_qr(Pc)
    out = {"kind": kind, "mm": mm, "bw": bw}
    res = {}
    for fast in (0, 1):
        R, Y, tau, T, usable, l2 = run(P0, fast)
        res[fast] = (R, Y, tau, T)
        nm = "fast" if fast else "exact"
        out[nm] = {
            "errR": float(np.linalg.norm(R - Pc) / np.linalg.norm(P0)),
            "errY": float(np.linalg.norm(Y - Yo) / max(np.linalg.norm(Yo), 1e-300)),
            "errtau": float(np.max(np.abs(tau - to))) if to.size else 0.0,
            "usable": int(usable), "l2": int(l2),
            "us": round(timed(P0, fast), 1),
        }
    out["bitwise_same"] = bool(all(np.array_equal(a, b) for a, b in zip(res[0], res[1])))
    print(json.dumps(out), flush=True)
lib.rq_set_option(h, b"fast_panel", 1)
