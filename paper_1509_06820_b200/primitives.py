"""Per-kernel entry points on CUDA tensors (column-major FP64), mirroring the
reference primitives one by one for parity tests and callers that drive the
block loop themselves:

  gemm            -> numpy matmul call sites (randomized.py:76,172-178; truncated.py:59,121,144-155)
  select_pivots   -> randomized.select_pivots (randomized.py:85-104)
  panel_qr        -> qrcp.panel_householder + randomized._panel_rank + kernels.build_t_matrix
  sample_update   -> randomized.sample_update (randomized.py:107-135)
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _abi
from .device import fmat, handle, is_fortran, ld, lib, ptr, stream_ptr


def _need_f(t, name):
    if not (torch.is_tensor(t) and t.is_cuda and t.dtype == torch.float64 and is_fortran(t)):
        raise ValueError(f"{name} must be a column-major float64 CUDA tensor")


def gemm(A, B, C_=None, alpha=1.0, beta=0.0, transa=False, transb=False):
    """C = alpha op(A) op(B) + beta C on the FP64 DMMA kernel."""
    _need_f(A, "A")
    _need_f(B, "B")
    m = A.shape[1] if transa else A.shape[0]
    k = A.shape[0] if transa else A.shape[1]
    n = B.shape[0] if transb else B.shape[1]
    kb = B.shape[1] if transb else B.shape[0]
    if k != kb:
        raise ValueError("inner dimensions differ")
    dev = A.device
    if C_ is None:
        C_ = fmat(m, n, dev, fill=0.0)
    _need_f(C_, "C")
    _abi.check(lib().rq_gemm(handle(dev), int(transa), int(transb), m, n, k, alpha, ptr(A), ld(A),
                             ptr(B), ld(B), beta, ptr(C_), ld(C_), stream_ptr(dev)))
    return C_


def select_pivots(B, want):
    """Returns (S pivoted transformed sample, piv list, got, Ys, taus, level2)."""
    _need_f(B, "B")
    ell, nt = B.shape
    dev = B.device
    S = fmat(ell, nt, dev, fill=0.0)
    piv = torch.zeros(max(want, 1), dtype=torch.int64, device=dev)
    Ys = fmat(ell, want, dev, fill=0.0)
    taus = torch.zeros(max(want, 1), dtype=torch.float64, device=dev)
    got = C.c_int64()
    l2 = C.c_int64()
    _abi.check(lib().rq_select_pivots(handle(dev), ell, nt, want, ptr(B), ld(B), ptr(S), ld(S),
                                      ptr(piv), ptr(Ys), ld(Ys), ptr(taus), C.byref(got),
                                      C.byref(l2), stream_ptr(dev)))
    g = int(got.value)
    return S, piv[:g].cpu().tolist(), g, Ys[:, :g], taus[:g], int(l2.value)


def panel_qr(P, tol=-1.0, with_t=True):
    """In-place panel QR of a column-major CUDA tensor; returns (Y, tau, T, usable, level2)."""
    _need_f(P, "P")
    mm, bw = P.shape
    dev = P.device
    Y = fmat(mm, bw, dev, fill=0.0)
    tau = torch.zeros(bw, dtype=torch.float64, device=dev)
    T = fmat(bw, bw, dev, fill=0.0) if with_t else None
    usable = C.c_int64()
    l2 = C.c_int64()
    _abi.check(lib().rq_panel_qr(handle(dev), mm, bw, ptr(P), ld(P), ptr(Y), ld(Y), ptr(tau),
                                 ptr(T), ld(T) if T is not None else 0, tol, C.byref(usable),
                                 C.byref(l2), stream_ptr(dev)))
    return Y, tau, T, int(usable.value), int(l2.value)


def sample_update(S, b, R11, R12, frob):
    """Returns (Bnew, degenerate)."""
    for t, nm in ((S, "S"), (R11, "R11"), (R12, "R12")):
        _need_f(t, nm)
    ell, ntot = S.shape
    n2 = ntot - b
    dev = S.device
    R = torch.cat([R11, R12], dim=1)
    Rf = fmat(R.shape[0], R.shape[1], dev)
    Rf.copy_(R)
    Bn = fmat(ell, n2, dev, fill=0.0)
    deg = C.c_int32()
    _abi.check(lib().rq_sample_update(handle(dev), ell, b, n2, ptr(S), ld(S), ptr(Rf),
                                      C.c_void_p(Rf.data_ptr() + 8 * b * ld(Rf)), ld(Rf), frob,
                                      ptr(Bn), ld(Bn), C.byref(deg), stream_ptr(dev)))
    return Bn, bool(deg.value)
