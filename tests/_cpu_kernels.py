"""CPU test doubles of the four GPU primitives the column-block-cyclic driver
calls (paper_1509_06820_b200.primitives: gemm, select_pivots, panel_qr,
sample_update), built on the oracle (oracle/port.py).  Test infrastructure
only: they let tests/test_parallel_gloo.py run the whole multi-rank control
flow of parallel.rqrcp_sharded on CPU ranks (gloo), where no GPU exists."""

import numpy as np
import torch

from oracle import port


def _np(t):
    return t.detach().cpu().numpy()


def _t(a):
    return torch.from_numpy(np.asfortranarray(np.asarray(a, dtype=np.float64)))


def gemm(A, B, C_=None, alpha=1.0, beta=0.0, transa=False, transb=False):
    a = _np(A).T if transa else _np(A)
    b = _np(B).T if transb else _np(B)
    if C_ is None or beta == 0.0:
        res = a @ b if alpha == 1.0 else alpha * (a @ b)
    elif alpha == -1.0 and beta == 1.0:
        res = _np(C_) - a @ b              # numpy's C - Y @ X (randomized.py:174-178)
    else:
        res = alpha * (a @ b) + beta * _np(C_)
    if C_ is None:
        return _t(res)
    C_.copy_(torch.from_numpy(res))
    return C_


def select_pivots(B, want):
    smp = port.Sample(B=np.asfortranarray(_np(B).copy()), ell=B.shape[0])
    ctr = port.Counters()
    perm, got = port.pick_pivots(smp, want, ctr)
    piv = [int(p) for _, p in perm.swaps[:got]]
    return _t(smp.B), piv, got, _t(smp.Ys), _t(smp.taus), ctr.level2_flops


def panel_qr(P, tol=-1.0, with_t=True):
    Pn = np.asfortranarray(_np(P).copy())
    ctr = port.Counters()
    Y, tau = port.panel_qr(Pn, ctr)
    usable = port.usable_columns(Pn, tol) if tol >= 0 else Pn.shape[1]
    T = port.t_factor(Y, tau) if with_t else None
    P.copy_(torch.from_numpy(Pn))
    return _t(Y), _t(tau), (_t(T) if T is not None else None), usable, ctr.level2_flops


def sample_update(S, b, R11, R12, frob):
    Sn = _np(S)
    smp = port.Sample(B=Sn, ell=Sn.shape[0], frob_a=frob)
    smp.s11, smp.s12, smp.s22 = Sn[:b, :b], Sn[:b, b:], Sn[b:, b:]
    try:
        port.downdate_sample(smp, _np(R11), _np(R12), port.Counters())
    except port.Degenerate:
        return None, True
    return _t(smp.B), False
