"""Unpivoted blocked QR and the presorted baseline on the GPU.

Drop-ins for the reference's qrcp.py:222-268 (``qr_blocked``,
``qr_presorted``) and kernels.py:184-186 (``column_norms``), with the same
signatures, validation and ``Factorization`` results.  The arithmetic runs in
librqrcp_b200.so: the panels and compact-WY block reflections of
``rq_qr_blocked`` (csrc/driver.cu) and the bit-exact column norms of
``rq_column_norms`` (csrc/small.cu).  There is no CPU fallback.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi
from .device import handle, ld, lib, ptr, require_cuda, stream_ptr, to_device_fortran
from .factorization import BlockReflectors, Factorization, OpCounters, Permutation
from .randomized import _validate_rank
from .truncated import qr_blocked_device


def _device_input(A):
    """(device F-order copy, True if the caller's array is a C-order host
    array -- numpy's axis-0 norm then sums rows in order)."""
    if torch.is_tensor(A) and A.is_cuda:
        return to_device_fortran(A, A.device), False
    a = np.asarray(A.cpu().numpy() if torch.is_tensor(A) else A, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-d array")
    seq = bool(a.flags.c_contiguous and not a.flags.f_contiguous)
    return to_device_fortran(a, require_cuda()), seq


def _column_norms_dev(Ad, sequential):
    m, n = Ad.shape
    out = torch.empty(max(n, 1), dtype=torch.float64, device=Ad.device)
    if n:
        _abi.check(lib().rq_column_norms(handle(Ad.device), ptr(Ad), m, n, ld(Ad),
                                         1 if sequential else 0, ptr(out), stream_ptr(Ad.device)))
    return out[:n]


def column_norms(A):
    """2-norms of the columns (kernels.py:184-186), bit-identical to
    ``np.linalg.norm(A, axis=0)`` for the caller's memory layout."""
    host = not (torch.is_tensor(A) and A.is_cuda)
    Ad, seq = _device_input(A)
    out = _column_norms_dev(Ad, seq)
    return out.cpu().numpy() if host else out


def _qr_blocked_dev(Ad, k, b, counters):
    """rq_qr_blocked on a private F-order copy: (Y, tau, work) with
    R = work[:k, :] and the trailing block work[k:, k:]."""
    import ctypes as C
    from .device import fmat
    m, n = Ad.shape
    work = fmat(m, n, Ad.device)
    work.copy_(Ad)
    Y = fmat(m, k, Ad.device)
    tau = torch.empty(max(k, 1), dtype=torch.float64, device=Ad.device)
    cnt = (C.c_int64 * 3)(0, 0, 0)
    _abi.check(lib().rq_qr_blocked(handle(Ad.device), m, n, k, b, ptr(work), ld(work), ptr(Y),
                                   ld(Y), ptr(tau), cnt, stream_ptr(Ad.device)))
    counters.gemm_flops += cnt[0]
    counters.level2_flops += cnt[1]
    counters.bytes_touched += cnt[2]
    return Y, tau[:k], work


def _result(Y, tau, work, k, perm, counters, host):
    R, trailing = work[:k, :], work[k:, k:]
    if host:
        Y, tau, R, trailing = (t.cpu().numpy() for t in (Y, tau, R, trailing))
    else:
        R, trailing = R.clone(), trailing.clone()
    return Factorization(reflectors=BlockReflectors(Y, tau), R=R, perm=perm, rank=k,
                         counters=counters, trailing=trailing)


def _checked(Ad, k, b, counters):
    m, n = Ad.shape
    k = _validate_rank(k, m, n)
    if b < 1:
        raise ValueError("block size must be >= 1")
    return k, counters if counters is not None else OpCounters()


def qr_blocked(A, k=None, b=32, counters=None):
    """Unpivoted blocked QR (qrcp.py:222-252): panel Householder QR plus one
    compact-WY reflection of the trailing matrix per block."""
    host = not (torch.is_tensor(A) and A.is_cuda)
    Ad, _ = _device_input(A)
    k, counters = _checked(Ad, k, b, counters)
    Y, tau, work = _qr_blocked_dev(Ad, k, b, counters)
    return _result(Y, tau, work, k, Permutation.identity(Ad.shape[1]), counters, host)


def qr_presorted(A, k=None, b=32, counters=None):
    """Blocked QR after a stable descending sort of the initial column norms
    (qrcp.py:255-268)."""
    host = not (torch.is_tensor(A) and A.is_cuda)
    Ad, seq = _device_input(A)
    k, counters = _checked(Ad, k, b, counters)
    order = torch.argsort(-_column_norms_dev(Ad, seq), stable=True)
    Y, tau, work = _qr_blocked_dev(Ad[:, order], k, b, counters)
    perm = Permutation.from_order(order.cpu().numpy())
    return _result(Y, tau, work, k, perm, counters, host)
