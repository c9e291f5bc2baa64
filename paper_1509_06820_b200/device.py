"""Tensor plumbing: PyTorch owns device memory and streams; the math runs in
librqrcp_b200.so.  Every matrix crossing the C-ABI is an FP64 column-major
(Fortran-order) CUDA tensor, i.e. shape (m, n) with strides (1, m)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1509_06820_b200 needs a CUDA (sm_100a) device; "
                           "there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise RuntimeError("paper_1509_06820_b200 runs on CUDA devices only")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


def fmat(rows, cols, device, fill=None):
    """Uninitialised (or filled) column-major FP64 matrix."""
    t = torch.empty((max(cols, 0), max(rows, 0)), dtype=torch.float64, device=device).t()
    if fill is not None:
        t.fill_(fill)
    return t


def is_fortran(t: torch.Tensor) -> bool:
    if t.dim() != 2:
        return False
    m, n = t.shape
    return t.stride(0) == 1 and (t.stride(1) >= max(m, 1) or n <= 1)


def ld(t: torch.Tensor) -> int:
    """Leading dimension of a column-major tensor."""
    m, n = t.shape
    return max(int(t.stride(1)) if n > 1 else m, 1)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def stream_ptr(device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def to_device_fortran(A, device) -> torch.Tensor:
    """Fresh column-major FP64 copy of A on `device` (the input is never mutated)."""
    if torch.is_tensor(A):
        src = A.detach()
        if src.dtype != torch.float64:
            src = src.to(torch.float64)
    else:
        arr = np.asarray(A, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("expected a 2-d array")
        src = torch.from_numpy(np.asfortranarray(arr))
    if src.dim() != 2:
        raise ValueError("expected a 2-d array")
    out = fmat(src.shape[0], src.shape[1], device)
    out.copy_(src, non_blocking=src.is_pinned() if not src.is_cuda else False)
    return out


def to_host(t: torch.Tensor | None):
    if t is None:
        return None
    return t.detach().cpu().numpy()


def lib():
    return _abi.load_library()


def handle(device: torch.device):
    return _abi.handle(device.index)
