"""Pivot selection on samples taller than 1024 rows against the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import port
from paper_1509_06820_b200.primitives import select_pivots
from paper_1509_06820_b200.device import to_device_fortran
dev = torch.device("cuda", 0)
for ell, nt, want in ((1000, 1500, 900), (1100, 1500, 1050), (1500, 3000, 1400), (2100, 2600, 2048)):
    g = np.random.default_rng(ell)
    B = g.standard_normal((ell, nt)) * np.exp(g.uniform(-2, 2, nt))
    smp = port.Sample(B=np.asfortranarray(B.copy()), ell=ell)
    t = time.time(); perm, got = port.pick_pivots(smp, want, port.Counters()); to = time.time() - t
    t = time.time(); S, piv, got_d, *_ = select_pivots(to_device_fortran(B, dev), want); torch.cuda.synchronize(); tg = time.time() - t
    fwd = list(range(nt))
    for j, p in enumerate(piv):
        fwd[j], fwd[p] = fwd[p], fwd[j]
    print(ell, nt, want, "got", got_d, got, "perm equal", np.array_equal(fwd, perm.forward),
          "S err", np.linalg.norm(S.cpu().numpy() - smp.B) / np.linalg.norm(B), "oracle s", round(to, 2), "gpu s", round(tg, 3), flush=True)
