"""Print GPU-vs-reference diffs for every golden fixture (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests import _golden as G
import paper_1509_06820_b200 as P

for name in G.case_names():
    rec = G.load(name)
    A = G.matrix_of(rec)
    cfg = P.RandomizedConfig(block=int(rec["block"]), padding=int(rec["padding"]), seed=int(rec["seed"]))
    drv = str(rec["driver"])
    try:
        f = getattr(P, drv)(A, G.k_of(rec), cfg)
    except Exception as e:
        print(f"{name}: EXC {e!r}"); continue
    frob = np.linalg.norm(A)
    line = f"{name}: rank {f.rank}/{int(rec['rank'])}"
    if drv == "tuxv":
        sv = f.singular_values(); line += f" sv_rel {np.max(np.abs(sv-rec['sv'])/np.maximum(rec['sv'],1e-300)):.2e}"
        line += f" gemm {f.counters.gemm_flops-int(rec['gemm_flops'])} l2 {f.counters.level2_flops-int(rec['level2_flops'])}"
        print(line); continue
    c = f.counters
    line += f" dgemm {c.gemm_flops-int(rec['gemm_flops'])} dl2 {c.level2_flops-int(rec['level2_flops'])} dbytes {c.bytes_touched-int(rec['bytes_touched'])} res {c.resamples}/{int(rec['resamples'])}"
    pf = np.asarray(f.perm.forward); pr = rec["perm"]
    line += f" perm_eq {np.array_equal(pf, pr)} first_diff {int(np.argmax(pf!=pr)) if not np.array_equal(pf,pr) else -1}"
    sw = np.array(f.perm.swaps).reshape(-1,2)
    line += f" swaps_eq {sw.shape==rec['swaps'].shape and np.array_equal(sw, rec['swaps'])}"
    if "R" in rec and rec["R"].shape == f.R.shape:
        line += f" Rrel {np.linalg.norm(f.R-rec['R'])/max(np.linalg.norm(rec['R']),1e-300):.2e}"
        Rr = np.zeros_like(rec["R"]); Rr[:, rec["perm"]] = rec["R"]
        line += f" RPt_rel {np.linalg.norm(f.perm.restore(f.R)-Rr)/max(np.linalg.norm(Rr),1e-300):.2e}"
    elif "R" in rec:
        d = np.abs(np.diag(rec["R"])); eps = np.finfo(float).eps
        sig = int(np.sum(d > 1e3 * eps * frob))
        line += f" sig_rank {sig} perm_sig_eq {np.array_equal(pf[:sig], pr[:sig])} Rsig_rel {np.linalg.norm(f.R[:sig]-rec['R'][:sig])/np.linalg.norm(rec['R'][:sig]):.2e}"
    else:
        line += f" Rdiag_rel {np.max(np.abs(np.diag(f.R)-rec['R_diag'])/np.maximum(np.abs(rec['R_diag']),1e-300)):.2e}"
    print(line, flush=True)
