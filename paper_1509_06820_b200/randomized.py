"""Randomized column-pivoted QR -- drop-in for pkg/src/rqrcp/randomized.py.

Same entry points and signatures as the reference (``rqrcp``, ``rsrqrcp``,
``ssrqrcp``, ``RandomizedConfig``), plus the north_star extension
``omega=`` (explicit first Omega, ell x m; resamples continue the seeded
stream at position ell*m).  The block loop runs natively in
librqrcp_b200.so (csrc/driver.cu) on sm_100a kernels; this module only
validates arguments with the reference's error messages, moves data, and
supplies the host Omega stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .device import fmat, handle, ld, lib, ptr, require_cuda, stream_ptr, to_device_fortran
from .factorization import BlockReflectors, Factorization, OpCounters, Permutation
from .rng import RngState


@dataclass
class RandomizedConfig:
    """randomized.py:22-40."""

    block: int = 32
    padding: int = 8
    seed: int = 0

    def __post_init__(self):
        if self.block < 1:
            raise ValueError("block must be >= 1")
        if self.padding < 1:
            raise ValueError("padding must be >= 1")

    @property
    def ell(self):
        return self.block + self.padding


class DegenerateSampleError(RuntimeError):
    """randomized.py:43-45 (raised and handled inside the native driver)."""


def _validate_rank(k, m, n):
    """qrcp.py:87-94."""
    kmax = min(m, n)
    if k is None:
        return kmax
    k = int(k)
    if not 0 <= k <= kmax:
        raise ValueError(f"rank {k} outside [0, {kmax}]")
    return k


class _OmegaSource:
    """ctypes callback feeding the native driver from the host RngState."""

    def __init__(self, rng: RngState):
        self.rng = rng

        def fill(_user, rows, cols, dst):
            try:
                buf = np.ctypeslib.as_array(dst, shape=(int(rows) * int(cols),))
                self.rng.fill(buf)
                return 0
            except Exception:  # pragma: no cover - surfaced as an ABI error
                return 1

        self.fn = _abi.OMEGA_FN(fill)

    def native(self):
        """FactorArgs fields that let the library draw this stream itself
        (rq_omega_fill on the same Philox key and raw counter: the same
        values as ``fill``), so resample draws can be made ahead on a host
        thread without calling back into Python.  The RngState is not
        advanced (each factorization owns a fresh one)."""
        from .rng import THREADS
        return dict(omega_native=1, omega_threads=THREADS, omega_k0=self.rng._k0,
                    omega_k1=self.rng._k1, omega_raw=self.rng._raw)


def _shape_of(A):
    if torch.is_tensor(A):
        if A.dim() != 2:
            raise ValueError("expected a 2-d array")
        return int(A.shape[0]), int(A.shape[1])
    a = np.asarray(A)
    if a.ndim != 2:
        raise ValueError("expected a 2-d array")
    return int(a.shape[0]), int(a.shape[1])


def _prepare_omega(omega, ell, m, seed, dev):
    if omega is None:
        return None, RngState(seed)
    om = to_device_fortran(omega, dev)
    if tuple(om.shape) != (ell, m):
        raise ValueError(f"omega must be {ell} x {m}")
    return om, RngState(seed, position=ell * m)


def run_native(A, k, config, *, variant, ell, width, omega=None, speculate=True, device=None,
               host_out=None):
    """Shared body of every factorization entry point: returns the raw device
    outputs plus the library's result struct.  host_out (default: A is a host
    array) streams Y and R into pinned host buffers while the blocks commit."""
    m, n = _shape_of(A)
    dev = require_cuda(device if device is not None else
                       (A.device if torch.is_tensor(A) and A.is_cuda else None))
    if host_out is None:
        host_out = not (torch.is_tensor(A) and A.is_cuda)
    work = to_device_fortran(A, dev)
    Y = fmat(m, k, dev)
    tau = torch.empty(k, dtype=torch.float64, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    cap = 2 * k + 16
    swaps = torch.empty(2 * cap, dtype=torch.int64, device=dev)
    W = R = None
    if variant == _abi.RQ_TRQRCP:
        W = fmat(n, k, dev)
        R = fmat(k, n, dev)
    om, rng = _prepare_omega(omega, ell, m, config.seed, dev)
    src = _OmegaSource(rng)
    hY = hR = None
    if host_out:
        # column-major pinned buffers (torch's caching host allocator recycles them)
        hY = torch.empty((k, m), dtype=torch.float64, pin_memory=True).t()
        hR = torch.empty((n, k), dtype=torch.float64, pin_memory=True).t()
    args = _abi.FactorArgs(
        m=m, n=n, k=k, block=width, ell=ell, variant=variant, speculate=1 if speculate else 0,
        work=ptr(work), ldw=ld(work), Y=ptr(Y), ldy=ld(Y), tau=ptr(tau),
        W=ptr(W), ldW=ld(W) if W is not None else 0, R=ptr(R), ldR=ld(R) if R is not None else 0,
        perm=ptr(perm), swaps=ptr(swaps), swap_cap=cap, omega0=ptr(om), omega_fn=src.fn,
        **src.native(), omega_user=None, stream=stream_ptr(dev),
        host_Y=hY.data_ptr() if hY is not None else None, ldhY=m,
        host_R=hR.data_ptr() if hR is not None else None, ldhR=k)
    res = _abi.FactorResult()
    _abi.check(lib().rq_factor(handle(dev), C.byref(args), C.byref(res)))
    return dict(work=work, Y=Y, tau=tau, perm=perm, swaps=swaps, W=W, R=R, res=res,
                rng=rng, device=dev, hY=hY, hR=hR)


def _counters(res):
    return OpCounters(gemm_flops=int(res.gemm_flops), level2_flops=int(res.level2_flops),
                      bytes_touched=int(res.bytes_touched), resamples=int(res.resamples))


def to_host_many(*ts):
    """D2H of several device tensors into pinned host buffers (torch's caching
    host allocator recycles them across calls), one stream sync, numpy views;
    column-major layouts are kept (no host-side reshuffle)."""
    outs = []
    dev = next((t.device for t in ts if t is not None), None)
    for t in ts:
        if t is None:
            outs.append(None)
            continue
        if t.dim() == 2 and t.stride(0) == 1 and t.shape[1] > 1:
            h = torch.empty((t.shape[1], t.shape[0]), dtype=t.dtype, pin_memory=True).t()
        else:
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    if dev is not None:
        torch.cuda.current_stream(dev).synchronize()   # the stream the copies were issued on
    return tuple(None if h is None else h.numpy() for h in outs)


def _swap_list(swaps, n):
    pairs = swaps[: 2 * n].view(-1, 2).cpu().numpy()
    return [(int(a), int(b)) for a, b in pairs]


def package(out, host, trailing_update=True, truncated=False):
    """Shape raw outputs into the reference's result types."""
    res = out["res"]
    rank = int(res.rank)
    swaps = _swap_list(out["swaps"], int(res.nswaps))
    Y = out["Y"][:, :rank]
    tau = out["tau"][:rank]
    if truncated:
        R = out["R"][:rank, :]
        W = out["W"][:, :rank]
        trailing = None
    else:
        R = out["work"][:rank, :]
        W = None
        trailing = out["work"][rank:, rank:] if trailing_update else None
    perm = out["perm"]
    if host and out.get("hY") is not None:
        # Y and R were streamed into pinned host buffers during the factorization
        Y = out["hY"][:, :rank].numpy()
        R = out["hR"][:rank, :].numpy()
        tau, W, trailing, perm = to_host_many(tau, W, trailing, perm)
    elif host:
        Y, tau, R, W, trailing, perm = to_host_many(Y, tau, R, W, trailing, perm)
    else:
        R = R.clone()
        trailing = trailing.clone() if trailing is not None else None
    return rank, Y, tau, R, W, trailing, Permutation(forward=perm, swaps=swaps)


def _randomized_factor(A, k, config, ell, block_width, variant, trailing_update, omega):
    m, n = _shape_of(A)
    k = _validate_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    if ell > m:
        raise ValueError(f"sample rows {ell} exceed matrix rows {m}")
    host = not (torch.is_tensor(A) and A.is_cuda)
    out = run_native(A, k, config, variant=variant, ell=ell, width=block_width, omega=omega)
    rank, Y, tau, R, _, trailing, perm = package(out, host, trailing_update)
    return Factorization(reflectors=BlockReflectors(Y, tau), R=R, perm=perm, rank=rank,
                         counters=_counters(out["res"]), trailing=trailing)


def rqrcp(A, k=None, config=None, omega=None):
    """Randomized pivoted QR, sample downdated across blocks (randomized.py:269-281)."""
    config = config if config is not None else RandomizedConfig()
    return _randomized_factor(A, k, config, config.ell, config.block, _abi.RQ_RQRCP, True, omega)


SSRQRCP_MAX_K = 256     # widest panel the native driver factors in one block (driver.cu)
SSRQRCP_MAX_ELL = 4096  # rows of the pivot kernel's sample (select.cu)


def rsrqrcp(A, k=None, config=None, omega=None):
    """Fresh sketch before every block (randomized.py:284-296)."""
    config = config if config is not None else RandomizedConfig()
    return _randomized_factor(A, k, config, config.ell, config.block, _abi.RQ_RSRQRCP, True,
                              omega)


def ssrqrcp(A, k, config=None, omega=None):
    """One (k + padding)-row sketch selects all k pivots (randomized.py:299-313)."""
    config = config if config is not None else RandomizedConfig()
    k = int(k)
    if k + config.padding > SSRQRCP_MAX_ELL:
        raise NotImplementedError(
            f"ssrqrcp with k = {k}: the (k + padding)-row sample exceeds the pivot kernel's "
            f"{SSRQRCP_MAX_ELL} rows (the reference accepts any k)")
    if k > SSRQRCP_MAX_K:
        return _ssrqrcp_wide(A, k, config, omega)
    return _randomized_factor(A, k, config, k + config.padding, k, _abi.RQ_SSRQRCP, False, omega)


def _ssrqrcp_wide(A, k, config, omega):
    """ssrqrcp with k > SSRQRCP_MAX_K: the reference's single block
    (randomized.py:207-258 with block width k and no trailing update) driven
    from the host over the C-ABI kernels -- the (k + p)-row sketch
    (rq_sketch), k pivot steps on it (rq_select_pivots), the panel QR of the k
    chosen columns as a blocked QR (rq_qr_blocked, 64-column panels: the
    Householder QR of the column-by-column panel, to rounding), _panel_rank
    on its diagonal (randomized.py:150-155) with the resample branches, and
    the block reflection for the R rows (randomized.py:158-180).  Counters
    follow the reference's formulas (the panel's level-2 count is the
    column-by-column one)."""
    from .device import fmat
    from .factorization import t_factor
    from .rng import gaussian_matrix
    from .truncated import qr_blocked_device
    m, n = _shape_of(A)
    k = _validate_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    ell = k + config.padding
    if ell > m:
        raise ValueError(f"sample rows {ell} exceed matrix rows {m}")
    host = not (torch.is_tensor(A) and A.is_cuda)
    dev = A.device if not host else require_cuda()
    work = to_device_fortran(A, dev)
    ctr = OpCounters()
    fr = torch.empty(1, dtype=torch.float64, device=dev)
    _abi.check(lib().rq_frob_norm(handle(dev), ptr(work), m, n, ld(work), ptr(fr), stream_ptr(dev)))
    frob = float(fr[0])
    tol = np.finfo(np.float64).eps * frob
    rng = RngState(config.seed)
    first = [omega]

    def sketch():
        om = first[0]
        first[0] = None
        if om is None:
            return make_sample(work, ell, rng, ctr)
        rng.position = ell * m   # the explicit Omega replaces the first draw
        omd = to_device_fortran(om, dev)
        B = fmat(ell, n, dev)
        _abi.check(lib().rq_sketch(handle(dev), ell, m, n, ptr(omd), ld(omd), ptr(work), ld(work),
                                   ptr(B), ld(B), stream_ptr(dev)))
        ctr.gemm_flops += 2 * ell * m * n
        ctr.bytes_touched += 8 * (ell * m + m * n + ell * n)
        return SampleState(B=B, ell=ell)

    if omega is not None and not (torch.is_tensor(omega) and omega.is_cuda):
        omega = np.asarray(omega, dtype=np.float64)
        if omega.shape != (ell, m):
            raise ValueError(f"omega must be {ell} x {m}")
    smp = sketch()
    smp.frob_a = frob
    perm = Permutation.identity(n)
    resampled = False
    Y = tau = None
    bw = 0
    while True:
        local, got = select_pivots(smp, k, ctr)
        if got < k and not resampled:
            smp = sketch()
            smp.frob_a = frob
            ctr.resamples += 1
            resampled = True
            continue
        if got == 0:
            break
        for a_, c_ in local.swaps:          # _apply_local_swaps (randomized.py:138-147)
            perm.swap(a_, c_)
        work = work[:, torch.as_tensor(local.forward, device=dev)]
        work = to_device_fortran(work, dev)
        Yp, tp, Rp = qr_blocked_device(work[:, :got], None, 64)
        taus = tp.cpu().numpy()
        for j in range(got):               # panel_householder's apply_reflector counts
            if taus[j] != 0.0 and got - j - 1 > 0:
                ctr.level2_flops += 4 * (m - j) * (got - j - 1)
                ctr.bytes_touched += 16 * (m - j) * (got - j - 1)
        d = torch.diagonal(Rp[:, :got]).abs().cpu().numpy()
        bad = d <= tol
        usable = int(np.argmax(bad)) if bad.any() else got
        if usable < got and not resampled:
            smp = sketch()
            smp.frob_a = frob
            ctr.resamples += 1
            resampled = True
            continue
        bw = usable
        if bw:
            work[:bw, :bw] = Rp[:bw, :bw]
            work[bw:, :bw] = 0.0
            Y, tau = Yp[:, :bw], tp[:bw]
        break
    if bw and n > bw:
        # _block_stages without the trailing update: R12 = C[:b] - Y[:b] (T^T (Y^T C))
        from . import primitives as K
        Yb = to_device_fortran(Y, dev)
        T = t_factor(Yb, tau)
        C_ = to_device_fortran(work[:, bw:], dev)
        X = K.gemm(T, K.gemm(Yb, C_, transa=True), transa=True)
        R12 = to_device_fortran(work[:bw, bw:], dev)
        K.gemm(to_device_fortran(Yb[:bw], dev), X, R12, alpha=-1.0, beta=1.0)
        work[:bw, bw:] = R12
        nt2 = n - bw
        ctr.gemm_flops += 2 * m * bw * nt2 + bw * bw * nt2 + 2 * bw * bw * nt2
        ctr.bytes_touched += 8 * (m * nt2 + m * bw + bw * nt2)
    if not bw:
        Y = fmat(m, 0, dev)
        tau = torch.zeros(0, dtype=torch.float64, device=dev)
    R = work[:bw, :].clone()
    if host:
        Y, tau, R = (t.cpu().numpy() for t in (Y, tau, R))
        perm = Permutation(forward=np.asarray(perm.forward), swaps=perm.swaps)
    else:
        perm = Permutation(forward=torch.as_tensor(perm.forward, device=dev), swaps=perm.swaps)
    return Factorization(reflectors=BlockReflectors(Y, tau), R=R, perm=perm, rank=bw,
                         counters=ctr, trailing=None)


# ---------------------------------------------------------------- sample-level primitives
# The reference's per-block building blocks (randomized.py:48-135) with its
# signatures, for callers that drive the block loop themselves; each runs on
# the C-ABI kernels the native driver uses (rq_sketch, rq_select_pivots,
# rq_sample_update).  numpy in -> numpy out; CUDA tensors stay on the device.


@dataclass
class SampleState:
    """The sketch and the pieces of its partial factorization
    (randomized.py:48-66): after :func:`select_pivots` ``B`` holds the
    transformed sample in pivoted column order, ``s11``/``s12``/``s22`` view
    its blocks, ``reflectors`` are the sample-side Householder vectors and
    ``frob_a`` is the Frobenius norm of the matrix being factored."""

    B: object
    ell: int
    block: int = 0
    s11: object = None
    s12: object = None
    s22: object = None
    reflectors: BlockReflectors | None = None
    frob_a: float = 0.0


def _as_dev_f(x, dev):
    return to_device_fortran(x, dev) if not (torch.is_tensor(x) and x.is_cuda) else \
        (x if x.dtype == torch.float64 and x.dim() == 2 and x.stride(0) == 1 else
         to_device_fortran(x, dev))


def make_sample(A, ell, rng, counters=None):
    """Sketch B = Omega A with a fresh ell x m standard Gaussian Omega drawn
    from ``rng`` (randomized.py:69-82): the same host stream as the
    reference, the product on the FP64 tensor-core GEMM (rq_sketch)."""
    from .rng import gaussian_matrix
    host = not (torch.is_tensor(A) and A.is_cuda)
    dev = A.device if not host else require_cuda()
    Ad = _as_dev_f(A, dev)
    m, n = Ad.shape
    if ell < 1:
        raise ValueError("sample must have at least one row")
    om = to_device_fortran(gaussian_matrix(rng, ell, m), dev)
    B = fmat(ell, n, dev)
    _abi.check(lib().rq_sketch(handle(dev), ell, m, n, ptr(om), ld(om), ptr(Ad), ld(Ad), ptr(B),
                               ld(B), stream_ptr(dev)))
    fr = torch.empty(1, dtype=torch.float64, device=dev)
    _abi.check(lib().rq_frob_norm(handle(dev), ptr(Ad), m, n, ld(Ad), ptr(fr), stream_ptr(dev)))
    if counters is not None:
        counters.gemm_flops += 2 * ell * m * n
        counters.bytes_touched += 8 * (ell * m + m * n + ell * n)
    return SampleState(B=B.cpu().numpy() if host else B, ell=ell, frob_a=float(fr[0]))


def select_pivots(sample, b, counters=None):
    """b greedy steps of pivoted Householder elimination on the sample
    (randomized.py:85-104): returns (local Permutation over the sample's
    columns, pivots delivered) and leaves the transformed pivoted sample and
    its blocks in ``sample``."""
    B = sample.B
    ell, nt = B.shape
    if not 1 <= b <= min(ell, nt):
        raise ValueError(f"cannot select {b} pivots from a {ell} x {nt} sample")
    host = not (torch.is_tensor(B) and B.is_cuda)
    dev = B.device if not host else require_cuda()
    Bd = _as_dev_f(B, dev)
    S = fmat(ell, nt, dev, fill=0.0)
    piv = torch.zeros(b, dtype=torch.int64, device=dev)
    Ys = fmat(ell, b, dev, fill=0.0)
    taus = torch.zeros(b, dtype=torch.float64, device=dev)
    got, l2 = C.c_int64(), C.c_int64()
    _abi.check(lib().rq_select_pivots(handle(dev), ell, nt, b, ptr(Bd), ld(Bd), ptr(S), ld(S),
                                      ptr(piv), ptr(Ys), ld(Ys), ptr(taus), C.byref(got),
                                      C.byref(l2), stream_ptr(dev)))
    g = int(got.value)
    if counters is not None:
        # apply_reflector counts 4 m n level-2 flops and touches A twice
        # (16 m n bytes) per step: bytes = 4 x level-2 (kernels.py:47-56)
        counters.level2_flops += int(l2.value)
        counters.bytes_touched += 4 * int(l2.value)
    perm = Permutation.identity(nt)
    for j, p in enumerate(piv[:g].cpu().tolist()):
        perm.swap(j, int(p))
    out = S.cpu().numpy() if host else S
    Y, tau = Ys[:, :g], taus[:g]
    sample.B = out
    sample.reflectors = BlockReflectors(Y.cpu().numpy() if host else Y,
                                        tau.cpu().numpy() if host else tau)
    sample.s11 = out[:g, :g]
    sample.s12 = out[:g, g:]
    sample.s22 = out[g:, g:]
    return perm, g


def sample_update(sample, R11, R12, counters=None):
    """Downdate the sample past a completed block, B1 = S12 - S11 R11^{-1}
    R12 stacked over S22 (randomized.py:107-135); raises
    DegenerateSampleError when any |R11_jj| < eps^(3/4) * frob_a."""
    b = R11.shape[0]
    if sample.s11 is None or sample.s11.shape[0] != b:
        raise ValueError("sample has no matching factorization to downdate")
    host = not (torch.is_tensor(sample.B) and sample.B.is_cuda)
    dev = sample.B.device if not host else require_cuda()
    n2 = R12.shape[1]
    if n2 == 0:
        r = torch.as_tensor(np.asarray(R11) if not torch.is_tensor(R11) else R11,
                            dtype=torch.float64).diagonal().abs()
        if bool((r < np.finfo(np.float64).eps ** 0.75 * sample.frob_a).any()):
            raise DegenerateSampleError("block triangle numerically singular; sample must be "
                                        "re-sketched")
        sample.B = np.zeros((sample.ell, 0)) if host else fmat(sample.ell, 0, dev)
    else:
        Sd = _as_dev_f(sample.B, dev)
        R = fmat(b, b + n2, dev)
        R[:, :b] = torch.as_tensor(R11, dtype=torch.float64, device=dev)
        R[:, b:] = torch.as_tensor(R12, dtype=torch.float64, device=dev)
        Bn = fmat(sample.ell, n2, dev, fill=0.0)
        deg = C.c_int32()
        _abi.check(lib().rq_sample_update(handle(dev), sample.ell, b, n2, ptr(Sd), ld(Sd), ptr(R),
                                          C.c_void_p(R.data_ptr() + 8 * b * ld(R)), ld(R),
                                          float(sample.frob_a), ptr(Bn), ld(Bn), C.byref(deg),
                                          stream_ptr(dev)))
        if deg.value:
            raise DegenerateSampleError("block triangle numerically singular; sample must be "
                                        "re-sketched")
        if counters is not None:
            counters.gemm_flops += 3 * b * b * n2
            counters.bytes_touched += 8 * (b * b + b * n2 + b * b + b * n2 + b * n2)
        sample.B = Bn.cpu().numpy() if host else Bn
    sample.block += 1
    sample.s11 = sample.s12 = sample.s22 = None
    sample.reflectors = None
    return sample
