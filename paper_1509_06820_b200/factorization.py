"""Result types of the drop-in API (kernels.py:59-136, qrcp.py:27-60,
truncated.py:32-50, 187-205, counters.py:12-27 of the reference).

Arrays are numpy when the caller passed host data and torch CUDA tensors
(column-major) when the caller passed a CUDA tensor; the methods work on
both and keep the dense verification products (``q_factor``) on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .device import fmat, handle, ld, lib, ptr, require_cuda, stream_ptr, to_device_fortran


@dataclass
class OpCounters:
    """counters.py:12-27: GEMM vs level-2 flops (2 per FMA), coarse bytes,
    resamples -- evaluated with the reference's per-call-site formulas."""

    gemm_flops: int = 0
    level2_flops: int = 0
    bytes_touched: int = 0
    resamples: int = 0

    def touch(self, *arrays):
        for a in arrays:
            self.bytes_touched += 8 * int(np.prod(a.shape))

    def merge(self, other):
        self.gemm_flops += other.gemm_flops
        self.level2_flops += other.level2_flops
        self.bytes_touched += other.bytes_touched
        self.resamples += other.resamples


def _is_t(x):
    return torch.is_tensor(x)


@dataclass
class Permutation:
    """forward[i] = original index of the column now at position i
    (A P = A[:, forward]); ``swaps`` is the ordered transposition log."""

    forward: np.ndarray
    swaps: list = field(default_factory=list)

    @classmethod
    def identity(cls, n):
        return cls(forward=np.arange(n), swaps=[])

    @classmethod
    def from_order(cls, order):
        order = np.asarray(order)
        perm = cls.identity(len(order))
        where = {int(v): i for i, v in enumerate(perm.forward)}
        for i, target in enumerate(order):
            j = where[int(target)]
            if j != i:
                where[int(perm.forward[i])] = j
                where[int(target)] = i
            perm.swap(i, j)
        return perm

    @property
    def n(self):
        return len(self.forward)

    def swap(self, i, j):
        self.swaps.append((i, j))
        if i != j:
            self.forward[[i, j]] = self.forward[[j, i]]

    def apply(self, A):
        return A[:, self.forward]

    def matrix(self):
        if _is_t(self.forward):
            return torch.eye(self.n, dtype=torch.float64, device=self.forward.device)[:, self.forward]
        return np.eye(self.n)[:, self.forward]

    def restore(self, R):
        if _is_t(R):
            out = torch.zeros_like(R)
            out[:, self.forward] = R
            return out
        out = np.zeros_like(R)
        out[:, self.forward] = R
        return out


@dataclass
class BlockReflectors:
    """Q = I - Y T Y^T; W is TRQRCP's n x rank inner-product panel."""

    Y: np.ndarray
    tau: np.ndarray
    T: np.ndarray | None = None
    W: np.ndarray | None = None

    @property
    def width(self):
        return self.Y.shape[1]

    def t_matrix(self):
        if self.T is None:
            self.T = t_factor(self.Y, self.tau)
        return self.T


def _dev_of(x):
    return x.device if _is_t(x) and x.is_cuda else require_cuda()


def t_factor(Y, tau):
    """build_t_matrix (kernels.py:139-147) on the GPU."""
    dev = _dev_of(Y)
    Yd = to_device_fortran(Y, dev)
    td = torch.as_tensor(np.asarray(tau) if not _is_t(tau) else tau, dtype=torch.float64,
                         device=dev).contiguous()
    nb = Yd.shape[1]
    T = fmat(nb, nb, dev, fill=0.0)
    if nb:
        _abi.check(lib().rq_t_factor(handle(dev), ptr(Yd), ld(Yd), Yd.shape[0], nb, ptr(td),
                                     ptr(T), ld(T), stream_ptr(dev)))
    return T if _is_t(Y) else T.cpu().numpy()


def q_columns(Y, tau, cols, block=64):
    """Leading ``cols`` columns of I - Y T Y^T (qrcp.py:53-60), on the GPU."""
    dev = _dev_of(Y)
    Yd = to_device_fortran(Y, dev)
    td = torch.as_tensor(np.asarray(tau) if not _is_t(tau) else tau, dtype=torch.float64,
                         device=dev).contiguous()
    m, nref = Yd.shape
    Q = fmat(m, cols, dev)
    _abi.check(lib().rq_q_columns(handle(dev), m, nref, cols, ptr(Yd), ld(Yd), ptr(td), block,
                                  ptr(Q), ld(Q), stream_ptr(dev)))
    return Q if _is_t(Y) else Q.cpu().numpy()


@dataclass
class Factorization:
    """A P = Q R with Q = I - Y T Y^T (qrcp.py:27-50)."""

    reflectors: BlockReflectors
    R: np.ndarray
    perm: Permutation
    rank: int
    counters: OpCounters
    trailing: np.ndarray | None = None

    def q_factor(self, full=False):
        Y, tau = self.reflectors.Y, self.reflectors.tau
        return q_columns(Y, tau, Y.shape[0] if full else self.rank)

    def reconstruct(self):
        return self.q_factor() @ self.R


@dataclass
class TruncatedFactorization:
    """Leading-k pivoted QR, A P ~= Q(:, :rank) R (truncated.py:32-50)."""

    reflectors: BlockReflectors
    R: np.ndarray
    perm: Permutation
    rank: int
    counters: OpCounters

    def q_factor(self):
        return q_columns(self.reflectors.Y, self.reflectors.tau, self.rank)

    def reconstruct(self):
        return self.q_factor() @ self.R


@dataclass
class TuxvFactorization:
    """A ~= U X V^T (truncated.py:187-205)."""

    U: np.ndarray
    V: np.ndarray
    X: np.ndarray
    iterations: int
    rank: int
    counters: OpCounters

    def approx(self):
        return self.U @ (self.X @ self.V.T)

    def singular_values(self):
        d = self.X.diagonal() if _is_t(self.X) else np.diag(self.X)
        if _is_t(d):
            return torch.sort(d.abs(), descending=True).values
        return np.sort(np.abs(d))[::-1]
