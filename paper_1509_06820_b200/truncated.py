"""Truncated factorizations -- drop-in for pkg/src/rqrcp/truncated.py.

``trqrcp`` (truncated.py:70-174) and ``tuxv`` (truncated.py:208-252) run in
librqrcp_b200.so; ``lq_factor`` (truncated.py:177-184) is the GPU blocked QR
of Z^T.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi
from .device import fmat, handle, ld, lib, ptr, require_cuda, stream_ptr, to_device_fortran
from .factorization import (
    BlockReflectors,
    OpCounters,
    TruncatedFactorization,
    TuxvFactorization,
    q_columns,
)
from .randomized import (
    RandomizedConfig,
    _OmegaSource,
    _prepare_omega,
    _shape_of,
    _validate_rank,
    package,
    run_native,
)


def _counters(res):
    return OpCounters(gemm_flops=int(res.gemm_flops), level2_flops=int(res.level2_flops),
                      bytes_touched=int(res.bytes_touched), resamples=int(res.resamples))


def _check_truncated(A, k, config):
    m, n = _shape_of(A)
    k = _validate_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    if config.ell > m:
        raise ValueError(f"sample rows {config.ell} exceed matrix rows {m}")
    return m, n, k


def trqrcp(A, k, config=None, omega=None):
    """Leading k rows of a randomized pivoted QR without trailing updates."""
    config = config if config is not None else RandomizedConfig()
    m, n, k = _check_truncated(A, k, config)
    host = not (torch.is_tensor(A) and A.is_cuda)
    out = run_native(A, k, config, variant=_abi.RQ_TRQRCP, ell=config.ell, width=config.block,
                     omega=omega)
    rank, Y, tau, R, W, _, perm = package(out, host, truncated=True)
    return TruncatedFactorization(reflectors=BlockReflectors(Y, tau, W=W), R=R, perm=perm,
                                  rank=rank, counters=_counters(out["res"]))


def qr_blocked_device(A, k=None, b=32, counters=None):
    """Unpivoted blocked QR (qrcp.py:222-252) on the GPU; returns (Y, tau, R)."""
    dev = A.device if torch.is_tensor(A) and A.is_cuda else require_cuda()
    work = to_device_fortran(A, dev)
    m, n = work.shape
    k = _validate_rank(k, m, n)
    Y = fmat(m, k, dev)
    tau = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
    cnt = (C.c_int64 * 3)(0, 0, 0)
    _abi.check(lib().rq_qr_blocked(handle(dev), m, n, k, b, ptr(work), ld(work), ptr(Y), ld(Y),
                                   ptr(tau), cnt, stream_ptr(dev)))
    if counters is not None:
        counters.gemm_flops += cnt[0]
        counters.level2_flops += cnt[1]
        counters.bytes_touched += cnt[2]
    return Y, tau[:k], work[:k, :]


def lq_factor(Z, b=32, counters=None):
    """Z = L V^T with orthonormal V, via the blocked QR of Z^T."""
    host = not (torch.is_tensor(Z) and Z.is_cuda)
    Zt = (Z.t() if torch.is_tensor(Z) else np.asarray(Z, dtype=np.float64).T)
    Y, tau, R = qr_blocked_device(Zt, b=b, counters=counters)
    V = q_columns(Y, tau, Y.shape[1])
    L = R.t()
    if host:
        return L.cpu().numpy(), V.cpu().numpy()
    return L, V


def tuxv(A, k, config=None, j_max=1, svd_of_x=False, omega=None):
    """Approximate truncated SVD A ~= U X V^T from TRQRCP (truncated.py:208-252)."""
    if torch.is_tensor(A):
        if A.dim() != 2:
            raise ValueError("expected a 2-d array")
    else:
        A = np.asarray(A, dtype=np.float64)
    if j_max < 1:
        raise ValueError("j_max must be >= 1")
    config = config if config is not None else RandomizedConfig()
    m, n, k = _check_truncated(A, k, config)
    host = not (torch.is_tensor(A) and A.is_cuda)
    dev = require_cuda(A.device if not host else None)
    Ad = to_device_fortran(A, dev)
    work = Ad.clone()
    Y = fmat(m, k, dev)
    tau = torch.empty(k, dtype=torch.float64, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    cap = 2 * k + 16
    swaps = torch.empty(2 * cap, dtype=torch.int64, device=dev)
    W = fmat(n, k, dev)
    R = fmat(k, n, dev)
    U = fmat(m, k, dev)
    V = fmat(n, k, dev)
    X = fmat(k, k, dev)
    om, rng = _prepare_omega(omega, config.ell, m, config.seed, dev)
    src = _OmegaSource(rng)
    fa = _abi.FactorArgs(
        m=m, n=n, k=k, block=config.block, ell=config.ell, variant=_abi.RQ_TRQRCP, speculate=1,
        work=ptr(work), ldw=ld(work), Y=ptr(Y), ldy=ld(Y), tau=ptr(tau), W=ptr(W), ldW=ld(W),
        R=ptr(R), ldR=ld(R), perm=ptr(perm), swaps=ptr(swaps), swap_cap=cap, omega0=ptr(om),
        omega_fn=src.fn, **src.native(), omega_user=None, stream=stream_ptr(dev))
    ta = _abi.TuxvArgs(f=fa, A=ptr(Ad), lda=ld(Ad), j_max=j_max, U=ptr(U), ldu=ld(U), V=ptr(V),
                       ldv=ld(V), X=ptr(X), ldx=ld(X))
    res = _abi.TuxvResult()
    _abi.check(lib().rq_tuxv(handle(dev), C.byref(ta), C.byref(res)))
    r = int(res.rank)
    U, V, X = U[:, :r], V[:, :r], X[:r, :r]
    if svd_of_x:
        # the k x k core's SVD (the reference uses its desk-scale Jacobi
        # oracle, svd.py:45-105, out of scope here): rotate U and V
        Ux, sx, Vxt = torch.linalg.svd(X)
        U = U @ Ux
        V = V @ Vxt.T
        X = torch.diag(sx)
    counters = _counters(res.f)
    if host:
        from .randomized import to_host_many
        U, V, X = to_host_many(U, V, X)
    else:
        U, V, X = U.clone(), V.clone(), X.clone()
    return TuxvFactorization(U=U, V=V, X=X, iterations=j_max, rank=r, counters=counters)
