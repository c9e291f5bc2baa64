"""Householder, WY-block and norm-bookkeeping primitives with the reference's
signatures (kernels.py:17-233 of the reference package), backed by the C-ABI:

  form_reflector          -> rq_panel_qr on a one-column panel
  apply_reflector         -> two rq_gemm calls (w = v^T A, A -= tau v w)
  compose_blocks          -> rq_gemm (T12 = -T1 (Y1^T Y2) T2)
  apply_block_reflection  -> three rq_gemm calls (W = Y^T A, W = T W, A -= Y W)
  downdate_norms          -> rq_downdate_norms (bit-identical to numpy)
  NormTracker             -> rq_column_norms + rq_downdate_norms

Arguments may be numpy arrays (results come back as numpy, in-place updates
are written back into the caller's array) or CUDA tensors (everything stays
on the device).  Counters follow the reference formulas exactly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .device import fmat, handle, is_fortran, ld, lib, ptr, require_cuda, stream_ptr
from .device import to_device_fortran
from .factorization import BlockReflectors, OpCounters, Permutation, t_factor  # noqa: F401
from .qrcp import column_norms

EPS = np.finfo(np.float64).eps
build_t_matrix = t_factor


def _is_dev(x):
    return torch.is_tensor(x) and x.is_cuda


def _dev(*xs):
    for x in xs:
        if _is_dev(x):
            return x.device
    return require_cuda()


def _fortran(x, dev):
    """Column-major FP64 device view of x: the tensor itself when it already
    is one, else a copy."""
    if _is_dev(x) and x.dtype == torch.float64 and is_fortran(x):
        return x
    return to_device_fortran(x, dev)


def _gemm(A, B, Cm, alpha=1.0, beta=0.0, ta=False, tb=False):
    m = A.shape[1] if ta else A.shape[0]
    k = A.shape[0] if ta else A.shape[1]
    n = B.shape[0] if tb else B.shape[1]
    dev = Cm.device
    _abi.check(lib().rq_gemm(handle(dev), int(ta), int(tb), m, n, k, alpha, ptr(A), ld(A),
                             ptr(B), ld(B), beta, ptr(Cm), ld(Cm), stream_ptr(dev)))
    return Cm


def _write_back(dst, src_dev):
    """In-place semantics for the caller's array."""
    if _is_dev(dst):
        if dst.data_ptr() != src_dev.data_ptr():
            dst.copy_(src_dev)
    else:
        dst[...] = src_dev.cpu().numpy()
    return dst


@dataclass
class Reflector:
    """Single Householder transform H = I - tau v v^T with v[0] = 1
    (kernels.py:17-23)."""

    v: np.ndarray
    tau: float
    beta: float


def form_reflector(x):
    """Reflector sending x to beta e1, beta = -sign(x[0]) ||x||, sign(0) = +1;
    a zero input yields the identity reflector (kernels.py:26-44).  One
    column of the panel kernel (csrc/panel.cu), which uses that convention."""
    host = not _is_dev(x)
    xs = np.asarray(x, dtype=np.float64) if host else x
    if xs.numel() == 0 if not host else xs.size == 0:
        raise ValueError("form_reflector needs a nonempty vector")
    dev = _dev(x)
    m = int(xs.shape[0])
    P = fmat(m, 1, dev)
    P.copy_(torch.as_tensor(xs, dtype=torch.float64, device=dev).reshape(m, 1))
    Y = fmat(m, 1, dev, fill=0.0)
    tau = torch.zeros(1, dtype=torch.float64, device=dev)
    usable, l2 = C.c_int64(), C.c_int64()
    _abi.check(lib().rq_panel_qr(handle(dev), m, 1, ptr(P), ld(P), ptr(Y), ld(Y), ptr(tau),
                                 None, 0, -1.0, C.byref(usable), C.byref(l2), stream_ptr(dev)))
    v = Y[:, 0]
    beta = float(P[0, 0])
    t = float(tau[0])
    return Reflector(v=v.cpu().numpy() if host else v.clone(), tau=t, beta=beta)


def apply_reflector(A, v, tau, counters=None):
    """In place A <- (I - tau v v^T) A (kernels.py:47-56)."""
    if A.shape[1] == 0 or tau == 0.0:
        return A
    dev = _dev(A, v)
    Ad = _fortran(A, dev)
    m, n = Ad.shape
    vd = _fortran(torch.as_tensor(v, dtype=torch.float64).reshape(m, 1) if not _is_dev(v)
                  else v.reshape(m, 1), dev)
    w = fmat(1, n, dev)
    _gemm(vd, Ad, w, ta=True)                        # w = v^T A
    _gemm(vd, w, Ad, alpha=-float(tau), beta=1.0)    # A -= tau v w
    if counters is not None:
        counters.level2_flops += 4 * m * n
        counters.bytes_touched += 2 * 8 * m * n
    return _write_back(A, Ad)


def compose_blocks(Y1, T1, Y2, T2):
    """WY form of (I - Y1 T1 Y1^T)(I - Y2 T2 Y2^T) (kernels.py:150-163)."""
    if Y2.shape[1] == 0:
        return Y1, T1
    if Y1.shape[1] == 0:
        return Y2, T2
    if Y1.shape[0] != Y2.shape[0]:
        raise ValueError("blocks must share a row count")
    host = not _is_dev(Y1)
    dev = _dev(Y1, T1, Y2, T2)
    y1, t1, y2, t2 = (_fortran(a, dev) for a in (Y1, T1, Y2, T2))
    b1, b2 = y1.shape[1], y2.shape[1]
    G = fmat(b1, b2, dev)
    _gemm(y1, y2, G, ta=True)                 # Y1^T Y2
    GT = fmat(b1, b2, dev)
    _gemm(G, t2, GT)                          # (Y1^T Y2) T2
    T = fmat(b1 + b2, b1 + b2, dev, fill=0.0)
    T[:b1, :b1] = t1
    T[b1:, b1:] = t2
    T12 = fmat(b1, b2, dev)
    _gemm(t1, GT, T12, alpha=-1.0)            # -T1 ((Y1^T Y2) T2)
    T[:b1, b1:] = T12
    Y = fmat(y1.shape[0], b1 + b2, dev)
    Y[:, :b1] = y1
    Y[:, b1:] = y2
    if host:
        return Y.cpu().numpy(), T.cpu().numpy()
    return Y, T


def apply_block_reflection(A, Y, T, transpose=False, counters=None):
    """In place A <- (I - Y T Y^T) A, or with T^T (kernels.py:166-181); the
    GEMM counter grows by exactly 4 m b n + b^2 n."""
    m, b = Y.shape
    n = A.shape[1]
    if b == 0 or n == 0:
        return A
    if A.shape[0] != m:
        raise ValueError(f"row mismatch: A has {A.shape[0]} rows, Y has {m}")
    dev = _dev(A, Y, T)
    Ad = _fortran(A, dev)
    Yd, Td = _fortran(Y, dev), _fortran(T, dev)
    W = fmat(b, n, dev)
    _gemm(Yd, Ad, W, ta=True)                 # W = Y^T A
    W2 = fmat(b, n, dev)
    _gemm(Td, W, W2, ta=bool(transpose))      # W = T W (or T^T W)
    _gemm(Yd, W2, Ad, alpha=-1.0, beta=1.0)   # A -= Y W
    if counters is not None:
        counters.gemm_flops += 4 * m * b * n + b * b * n
        counters.bytes_touched += 8 * (2 * m * n + m * b + b * n)
    return _write_back(A, Ad)


def _downdate_dev(nd, rd, inc, orig=None, guard=0.0, out=None):
    dev = nd.device
    n = int(nd.shape[0])
    out = nd if out is None else out
    flags = torch.zeros(max(n, 1), dtype=torch.int32, device=dev) if orig is not None else None
    if n:
        _abi.check(lib().rq_downdate_norms(handle(dev), ptr(nd), ptr(rd), inc, n,
                                           ptr(orig) if orig is not None else None, guard,
                                           ptr(out), ptr(flags) if flags is not None else None,
                                           stream_ptr(dev)))
    return out, (flags[:n] if flags is not None else None)


def _vec_dev(x, dev):
    t = torch.as_tensor(np.asarray(x, dtype=np.float64) if not torch.is_tensor(x) else x,
                        dtype=torch.float64, device=dev)
    return t.contiguous() if t.dim() == 1 else t.reshape(-1).contiguous()


def downdate_norms(norms, row):
    """Column norms after removing one row's contribution, clipped at zero
    (kernels.py:189-192); bit-identical to the reference."""
    host = not _is_dev(norms)
    dev = _dev(norms, row)
    nd = _vec_dev(norms, dev)
    rd = _vec_dev(row, dev)
    if rd.shape[0] != nd.shape[0]:
        raise ValueError("norms and row differ in length")
    out = torch.empty_like(nd)
    _downdate_dev(nd, rd, 1, out=out)
    return out.cpu().numpy() if host else out


class NormTracker:
    """Trailing column norms maintained by downdating, with the sqrt(eps)
    recompute guard (kernels.py:196-233).  The norms live on the device; a
    numpy input gets numpy views back from ``norms``/``max_trailing``."""

    GUARD = np.sqrt(EPS)

    def __init__(self, A):
        self._host = not _is_dev(A)
        norms = column_norms(A)                              # bit-identical to numpy
        self._dev = _dev(A)
        self._n = _vec_dev(norms, self._dev)
        self._orig = self._n * self._n                       # norms**2 (one rounding, as numpy)

    @property
    def norms(self):
        return self._n.cpu().numpy() if self._host else self._n

    @property
    def orig_sq(self):
        return self._orig.cpu().numpy() if self._host else self._orig

    def swap(self, i, j):
        if i != j:
            for t in (self._n, self._orig):
                t[[i, j]] = t[[j, i]]

    def max_trailing(self, start):
        """(position, norm) of the largest trailing norm; first max wins."""
        tail = self._n[start:].cpu().numpy()
        p = int(np.argmax(tail)) + start
        return p, float(tail[p - start])

    def downdate(self, start, row, materialize):
        """Remove ``row``'s contribution from columns start.. and recompute any
        column whose downdated norm is no longer trustworthy."""
        n = int(self._n.shape[0]) - start
        if n <= 0:
            return
        rd = _vec_dev(row, self._dev)
        tail = self._n[start:]
        _, unsafe = _downdate_dev(tail, rd, 1, orig=self._orig[start:], guard=float(self.GUARD),
                                  out=tail)
        for local in torch.nonzero(unsafe).flatten().tolist():
            c = start + int(local)
            col = materialize(c)
            fresh = column_norms(np.asarray(col, dtype=np.float64).reshape(-1, 1)
                                 if not _is_dev(col) else col.reshape(-1, 1))
            f = float(fresh[0])
            self._n[c] = f
            self._orig[c] = f * f
