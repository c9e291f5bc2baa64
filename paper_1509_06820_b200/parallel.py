"""Column-block-cyclic multi-GPU RQRCP.

Layout: global column position j lives on rank (j // b) % G at local index
(j // (b G)) b + j % b, where b is the pivot block width.  Per block J
(randomized.py:207-258 control flow, every branch decided identically on all
ranks because every decision input is replicated and every kernel is
deterministic):

1. every rank holds the full ell x nt sample and runs the pivot-selection
   kernel redundantly -> bitwise the same pivots everywhere;
2. the swaps (i0+j, i0+piv[j]) become one net permutation of the touched
   positions; columns whose source and destination ranks differ move with
   point-to-point sends (``exchange_columns``);
3. the owner of block-column J runs the panel kernel and broadcasts
   (usable, Y, tau, T, R11);
4. every rank updates ITS trailing columns: G = Y^T C, X = T^T G, C -= Y X;
5. R12 (b x nt) is all-gathered in position order and every rank applies the
   sample update redundantly (column-local math, replicated result).

Data movement uses ``torch.distributed`` (NCCL over NVLink on GPUs; the
exchange helpers are device-agnostic, so they are tested with gloo on CPU).
The math runs in librqrcp_b200.so through the same C-ABI primitives as the
single-GPU path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

EPS = float(np.finfo(np.float64).eps)


# ---------------------------------------------------------------- layout

@dataclass(frozen=True)
class BlockCyclic:
    """Column-block-cyclic map of n column positions over `world` ranks."""

    n: int
    b: int
    world: int

    def owner(self, j: int) -> int:
        return (j // self.b) % self.world

    def local_index(self, j: int) -> int:
        blk = j // self.b
        return (blk // self.world) * self.b + j % self.b

    def positions(self, rank: int) -> np.ndarray:
        """Global positions held by `rank`, in local order (cached)."""
        cache = self.__dict__.setdefault("_pos_cache", {})
        p = cache.get(rank)
        if p is None:
            j = np.arange(self.n)
            p = cache[rank] = j[(j // self.b) % self.world == rank]
        return p

    def n_local(self, rank: int) -> int:
        return int(self.positions(rank).size)

    def first_local_at_or_after(self, rank: int, pos: int) -> int:
        """Local index of the first column of `rank` whose position >= pos
        (local columns are in increasing position order, so the tail from
        here is contiguous)."""
        p = self.positions(rank)
        return int(np.searchsorted(p, pos))


def shard(A: np.ndarray, layout: BlockCyclic, rank: int) -> np.ndarray:
    """This rank's columns of A (host helper for setup and tests)."""
    return np.asfortranarray(np.asarray(A)[:, layout.positions(rank)])


# ---------------------------------------------------------------- swaps

def swap_plan(piv, got: int, i0: int) -> list[tuple[int, int]]:
    """Net effect of the ordered swaps (i0+j, i0+piv[j]), j < got
    (randomized.py:138-147), as moves (dst_position, src_position) with
    dst != src.  Applying every move simultaneously equals the sequence."""
    cur: dict[int, int] = {}
    for j in range(got):
        a, c = i0 + j, i0 + int(piv[j])
        if a == c:
            continue
        sa, sc = cur.get(a, a), cur.get(c, c)
        cur[a], cur[c] = sc, sa
    return [(d, s) for d, s in sorted(cur.items()) if d != s]


def exchange_columns(local: torch.Tensor, layout: BlockCyclic, moves, rank: int,
                     group=None) -> None:
    """Apply a column permutation (dst <- src moves over global positions) to
    the distributed matrix in place.  Columns whose source and destination
    ranks differ are packed per peer and moved with one send/recv pair each.
    Columns are gathered / scattered with one index kernel per batch on the
    transposed (row-contiguous) view of the column-major local block."""
    if not moves:
        return
    world = layout.world
    li = layout.local_index
    owner = layout.owner
    rows = local.t()                       # (n_local x m), each row = one local column
    dev = local.device
    # snapshot every source column this rank owns before anything is overwritten
    mine_src = sorted({s for _, s in moves if owner(s) == rank})
    slot = {s: k for k, s in enumerate(mine_src)}
    snap = rows.index_select(0, torch.as_tensor([li(s) for s in mine_src], device=dev)) \
        if mine_src else None
    loc_dst, loc_src = [], []
    out_by_peer: dict[int, list[int]] = {}
    in_by_peer: dict[int, list[int]] = {}
    for d, s in moves:
        od, os_ = owner(d), owner(s)
        if od == rank and os_ == rank:
            loc_dst.append(li(d))
            loc_src.append(slot[s])
        elif os_ == rank:
            out_by_peer.setdefault(od, []).append(slot[s])
        elif od == rank:
            in_by_peer.setdefault(os_, []).append(li(d))
    if loc_dst:
        rows.index_copy_(0, torch.as_tensor(loc_dst, device=dev),
                         snap.index_select(0, torch.as_tensor(loc_src, device=dev)))
    ops, recvbufs = [], []
    for peer in range(world):
        if peer == rank:
            continue
        if peer in out_by_peer:
            buf = snap.index_select(0, torch.as_tensor(out_by_peer[peer], device=dev))
            ops.append(dist.P2POp(dist.isend, buf, _grank(peer, group), group=group))
            recvbufs.append((None, buf))   # keep alive until the wait
        if peer in in_by_peer:
            buf = torch.empty((len(in_by_peer[peer]), local.shape[0]), dtype=local.dtype,
                              device=dev)
            recvbufs.append((peer, buf))
            ops.append(dist.P2POp(dist.irecv, buf, _grank(peer, group), group=group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for peer, buf in recvbufs:
        if peer is not None:
            rows.index_copy_(0, torch.as_tensor(in_by_peer[peer], device=dev), buf)


def _grank(r, group):
    return r if group is None else dist.get_global_rank(group, r)


# ---------------------------------------------------------------- gathers

def allgather_positions(local_tail: torch.Tensor, layout: BlockCyclic, pos0: int, rank: int,
                        group=None) -> torch.Tensor:
    """All-gather every rank's columns with position >= pos0 (its contiguous
    local tail) and assemble them in global position order: returns a
    (rows x (n - pos0)) tensor on every rank."""
    world = layout.world
    rows = local_tail.shape[0]
    if world == 1:
        return local_tail                 # the rank's tail is already in position order
    counts = [int(np.sum(layout.positions(r) >= pos0)) for r in range(world)]
    width = max(counts) if counts else 0
    pad = torch.zeros((rows, width), dtype=local_tail.dtype, device=local_tail.device)
    pad[:, : local_tail.shape[1]] = local_tail
    flat = pad.t().contiguous()                      # (width x rows), one column per row
    gathered = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(gathered, flat, group=group)
    out = torch.empty((rows, layout.n - pos0), dtype=local_tail.dtype, device=local_tail.device)
    cache = layout.__dict__.setdefault("_gather_idx", {})
    for r in range(world):
        key = (pos0, r, str(local_tail.device))
        idx = cache.get(key)
        if idx is None:
            p = layout.positions(r)
            p = p[p >= pos0] - pos0
            idx = cache[key] = torch.as_tensor(p, device=local_tail.device)
        if idx.numel():
            out[:, idx] = gathered[r][: idx.numel()].t()
    return out


def broadcast(t: torch.Tensor, src: int, group=None) -> torch.Tensor:
    """In-place broadcast; column-major matrices go through their (contiguous)
    transposed view, which shares the storage."""
    buf = t if t.is_contiguous() else t.t()
    if not buf.is_contiguous():
        raise ValueError("broadcast needs a dense row- or column-major tensor")
    dist.broadcast(buf, _grank(src, group), group=group)
    return t


def _panel(K, P, tol):
    """panel_householder + _panel_rank + build_t_matrix of the owner's panel
    (qrcp.py:206-219, randomized.py:150-155).  With the GPU kernels a 65..128
    column panel runs as two 64-column halves (the recursive panel QR the
    native driver uses: the first 64 reflectors from the first 64 columns,
    applied to the rest, whose rows below 64 are factored next, T = [[T1,
    -T1 (Y1^T Y2) T2], [0, T2]]), so both halves take the CholeskyQR2 fast
    path; a half that is not full rank falls back to the whole panel on the
    original columns, whose level-2 count and rank cut the reference defines."""
    mm, got = P.shape
    from . import primitives
    if K is not primitives or not 64 < got <= 128 or mm < got + 64:
        return K.panel_qr(P, tol=tol, with_t=True)
    from .device import fmat
    orig = fmat(mm, got, P.device)
    orig.copy_(P)
    h2 = got - 64
    P1 = P[:, :64]
    Y1, t1, T1, u1, l2a = K.panel_qr(P1, tol=tol, with_t=True)
    if u1 == 64:
        P2 = P[:, 64:]
        X = K.gemm(T1, K.gemm(Y1, P2, transa=True), transa=True)     # T1^T (Y1^T P2)
        K.gemm(Y1, X, P2, alpha=-1.0, beta=1.0)                       # P2 -= Y1 X
        Y2, t2, T2, u2, l2b = K.panel_qr(P[64:, 64:], tol=tol, with_t=True)
        if u2 == h2:
            Y = fmat(mm, got, P.device, fill=0.0)
            Y[:, :64] = Y1
            Y[64:, 64:] = Y2
            T = fmat(got, got, P.device, fill=0.0)
            T[:64, :64] = T1
            T[64:, 64:] = T2
            G = K.gemm(_f(Y1[64:]), Y2, transa=True)                    # Y1^T Y2 (rows >= 64)
            T[:64, 64:] = K.gemm(T1, K.gemm(G, T2), alpha=-1.0)
            # reflectors 1..64 applied to columns 65..got (apply_reflector counts)
            l2x = 4 * sum((mm - j) * h2 for j in range(64))
            return Y, torch.cat([t1, t2]), T, got, l2a + l2b + l2x
    P.copy_(orig)
    return K.panel_qr(P, tol=tol, with_t=True)


# ---------------------------------------------------------------- driver

@dataclass
class ShardedFactorization:
    """Result of `rqrcp_sharded`: replicated reflectors/permutation, this
    rank's R columns (``R_local``) and, when gathered, the full R."""

    Y: torch.Tensor
    tau: torch.Tensor
    perm: np.ndarray
    swaps: list
    rank: int
    R_local: torch.Tensor
    R: torch.Tensor | None = None
    layout: BlockCyclic | None = None
    counters: dict = field(default_factory=dict)


def rqrcp_sharded(A_local: torch.Tensor, m: int, n: int, k=None, config=None, group=None,
                  gather_r: bool = True, kernels=None) -> ShardedFactorization:
    """Full/partial RQRCP of the column-block-cyclic distributed A
    (randomized.py:183-266 semantics) on the ranks of `group`, one GPU each.

    `kernels` supplies gemm / select_pivots / panel_qr / sample_update with
    the signatures of paper_1509_06820_b200.primitives (the default, the
    sm_100a kernels); the CPU multi-rank tests pass oracle-backed doubles."""
    from . import primitives
    from .device import fmat
    K = kernels if kernels is not None else primitives
    from .randomized import RandomizedConfig, _validate_rank
    from .rng import RngState, gaussian_matrix

    config = config if config is not None else RandomizedConfig()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    b, ell = config.block, config.ell
    layout = BlockCyclic(n, b, world)
    k = _validate_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    if ell > m:
        raise ValueError(f"sample rows {ell} exceed matrix rows {m}")
    dev = A_local.device
    nloc = layout.n_local(me)
    work = fmat(m, nloc, dev)
    work.copy_(A_local)
    ss = (work * work).sum().reshape(1)
    dist.all_reduce(ss, group=group)
    frob = float(ss.sqrt().item())
    tol = EPS * frob
    rng = RngState(config.seed)
    Y = fmat(m, k, dev, fill=0.0)
    tau = torch.zeros(k, dtype=torch.float64, device=dev)
    perm = np.arange(n)
    swaps: list = []
    ctr = {"gemm_flops": 0, "level2_flops": 0, "resamples": 0}

    def sketch(i0: int) -> torch.Tensor:
        om = torch.from_numpy(gaussian_matrix(rng, ell, m - i0)).to(dev)
        lc = layout.first_local_at_or_after(me, i0)
        local = K.gemm(_f(om), _f(work[i0:, lc:]))          # ell x local tail
        ctr["gemm_flops"] += 2 * ell * (m - i0) * (n - i0)
        return _f(allgather_positions(local, layout, i0, me, group))

    B = sketch(0)
    rank_out = k
    i0 = 0
    while i0 < k:
        want = min(b, k - i0)
        owner = layout.owner(i0)
        resampled = False
        while True:
            S, piv, got, _, _, l2 = K.select_pivots(B, want)
            ctr["level2_flops"] += l2
            if got < want and not resampled:
                B = sketch(i0)
                ctr["resamples"] += 1
                resampled = True
                continue
            if got == 0:
                bw = 0
                break
            for j in range(got):
                a, c = i0 + j, i0 + piv[j]
                swaps.append((a, c))
                if a != c:
                    perm[a], perm[c] = perm[c], perm[a]
            exchange_columns(work, layout, swap_plan(piv, got, i0), me, group)
            meta = torch.zeros(2, dtype=torch.int64, device=dev)   # usable, panel level-2 flops
            lp = layout.local_index(i0)
            if me == owner:
                P = fmat(m - i0, got, dev)
                P.copy_(work[i0:, lp:lp + got])
                Yp, tp, T, usable, l2p = _panel(K, P, tol)
                meta[0], meta[1] = usable, l2p
            broadcast(meta, owner, group)
            usable = int(meta[0].item())
            ctr["level2_flops"] += int(meta[1].item())
            if usable < got and not resampled:
                B = sketch(i0)
                ctr["resamples"] += 1
                resampled = True
                continue
            bw = usable
            if bw:
                rows = max(m - i0, 2 * bw)
                blk = fmat(rows, 2 * bw + 1, dev) if me != owner else None
                if me == owner:
                    work[i0:, lp:lp + bw] = P[:, :bw]
                    # the leading bw x bw block of the panel's T is the T of
                    # its first bw reflectors (same T the native driver uses)
                    Tb = T[:bw, :bw]
                    blk = fmat(rows, 2 * bw + 1, dev, fill=0.0)
                    blk[: m - i0, :bw] = Yp[:, :bw]
                    blk[:bw, bw:2 * bw] = Tb
                    blk[:bw, 2 * bw] = tp[:bw]
                    blk[bw:2 * bw, bw:2 * bw] = P[:bw, :bw]      # R11 below T
                broadcast(blk, owner, group)
                Y[i0:, i0:i0 + bw] = blk[: m - i0, :bw]
                tau[i0:i0 + bw] = blk[:bw, 2 * bw]
                T = _f(blk[:bw, bw:2 * bw])
                R11 = _f(blk[bw:2 * bw, bw:2 * bw])
            break
        if bw == 0:
            rank_out = i0
            break
        # ---- block stages on my trailing columns (randomized.py:158-180)
        nt2 = n - i0 - bw
        lc = layout.first_local_at_or_after(me, i0 + bw)
        Yb = _f(Y[i0:, i0:i0 + bw])
        if nt2:
            C = work[i0:, lc:]
            if C.shape[1]:
                G = K.gemm(Yb, _f(C), transa=True)
                X = K.gemm(T, G, transa=True)
                K.gemm(Yb, X, C, alpha=-1.0, beta=1.0)
            mm = m - i0
            ctr["gemm_flops"] += (2 * mm * bw * nt2 + bw * bw * nt2 + 2 * bw * bw * nt2
                                  + (2 * (mm - bw) * bw * nt2 if i0 + bw < m else 0))
        i0 += bw
        if bw < want:
            rank_out = i0
            break
        if i0 < k:
            R12 = allgather_positions(_f(work[i0 - bw:i0, lc:]), layout, i0, me, group)
            Bn, degenerate = K.sample_update(S, bw, R11, _f(R12), frob)
            if degenerate:
                B = sketch(i0)
                ctr["resamples"] += 1
            else:
                B = Bn
                ctr["gemm_flops"] += 3 * bw * bw * (n - i0)
    R_local = work[:rank_out, :].clone()
    R = _f(allgather_positions(R_local, layout, 0, me, group)) if gather_r else None
    return ShardedFactorization(Y=Y[:, :rank_out], tau=tau[:rank_out], perm=perm, swaps=swaps,
                                rank=rank_out, R_local=R_local, R=R, layout=layout,
                                counters=ctr)



@dataclass
class ShardedTruncated:
    """Result of `trqrcp_sharded`: replicated Y, tau, permutation; this rank's
    columns of R (k x n) and rows of W (n x k, stored transposed as k x
    n_local, one column per position), and, when gathered, the full R and W."""

    Y: torch.Tensor
    tau: torch.Tensor
    perm: np.ndarray
    swaps: list
    rank: int
    R_local: torch.Tensor
    Wt_local: torch.Tensor
    R: torch.Tensor | None = None
    W: torch.Tensor | None = None
    layout: BlockCyclic | None = None
    counters: dict = field(default_factory=dict)


def trqrcp_sharded(A_local: torch.Tensor, m: int, n: int, k: int, config=None, group=None,
                   gather: bool = True, kernels=None) -> ShardedTruncated:
    """Truncated RQRCP (no trailing update) of the column-block-cyclic
    distributed A, truncated.py:70-174 semantics.  A is never modified: the
    rows of W and the columns of R follow A's columns (swapped together,
    truncated.py:114), Y is replicated.  Per block every rank forms its own
    columns of G = Y_b^T A - (Y_b^T Y) W^T, of W and of the new R rows; the
    owner of the block's columns forms and broadcasts the panel; R12 is
    all-gathered for the replicated sample update; a resample sketches each
    rank's columns implicitly (Omega A - (Omega Y) W^T, truncated.py:53-67)
    and all-gathers them."""
    from . import primitives
    from .device import fmat
    from .randomized import RandomizedConfig, _validate_rank
    from .rng import RngState, gaussian_matrix
    K = kernels if kernels is not None else primitives

    config = config if config is not None else RandomizedConfig()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    b, ell = config.block, config.ell
    layout = BlockCyclic(n, b, world)
    k = _validate_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    if ell > m:
        raise ValueError(f"sample rows {ell} exceed matrix rows {m}")
    dev = A_local.device
    nloc = layout.n_local(me)
    work = fmat(m, nloc, dev)
    work.copy_(A_local)
    ss = (work * work).sum().reshape(1)
    dist.all_reduce(ss, group=group)
    frob = float(ss.sqrt().item())
    tol = EPS * frob
    rng = RngState(config.seed)
    Y = fmat(m, k, dev, fill=0.0)
    tau = torch.zeros(k, dtype=torch.float64, device=dev)
    Wt = fmat(k, nloc, dev, fill=0.0)     # W^T: column = position
    R = fmat(k, nloc, dev, fill=0.0)
    perm = np.arange(n)
    swaps: list = []
    ctr = {"gemm_flops": 0, "level2_flops": 0, "resamples": 0}

    def sketch(i0: int) -> torch.Tensor:
        om = _f(torch.from_numpy(gaussian_matrix(rng, ell, m - i0)).to(dev))
        lc = layout.first_local_at_or_after(me, i0)
        local = K.gemm(om, _f(work[i0:, lc:]))                     # Omega A (my columns)
        ctr["gemm_flops"] += 2 * ell * (m - i0) * (n - i0)
        if i0:
            Z = K.gemm(om, _f(Y[i0:, :i0]))                         # Omega Y
            if local.shape[1]:
                K.gemm(Z, _f(Wt[:i0, lc:]), local, alpha=-1.0, beta=1.0)
            ctr["gemm_flops"] += 2 * ell * (m - i0) * i0 + 2 * ell * i0 * (n - i0)
        return _f(allgather_positions(local, layout, i0, me, group))

    B = sketch(0)
    rank_out = k
    i0 = 0
    while i0 < k:
        want = min(b, k - i0)
        owner = layout.owner(i0)
        lp = layout.local_index(i0)
        resampled = False
        while True:
            S, piv, got, _, _, l2 = K.select_pivots(B, want)
            ctr["level2_flops"] += l2
            if got < want and not resampled:
                B = sketch(i0)
                ctr["resamples"] += 1
                resampled = True
                continue
            if got == 0:
                bw = 0
                break
            for j in range(got):
                a, c = i0 + j, i0 + piv[j]
                swaps.append((a, c))
                if a != c:
                    perm[a], perm[c] = perm[c], perm[a]
            moves = swap_plan(piv, got, i0)
            for M_ in (work, Wt, R):                                # A's columns and followers
                exchange_columns(M_, layout, moves, me, group)
            meta = torch.zeros(2, dtype=torch.int64, device=dev)
            if me == owner:
                # materialise the selected columns: A[i0:, sel] - Y[i0:, :i0] W[sel, :i0]^T
                P = fmat(m - i0, got, dev)
                P.copy_(work[i0:, lp:lp + got])
                if i0:
                    K.gemm(_f(Y[i0:, :i0]), _f(Wt[:i0, lp:lp + got]), P, alpha=-1.0, beta=1.0)
                Yp, tp, T, usable, l2p = _panel(K, P, tol)
                meta[0], meta[1] = usable, l2p
            if i0:
                ctr["gemm_flops"] += 2 * (m - i0) * i0 * got
            broadcast(meta, owner, group)
            usable = int(meta[0].item())
            ctr["level2_flops"] += int(meta[1].item())
            if usable < got and not resampled:
                B = sketch(i0)
                ctr["resamples"] += 1
                resampled = True
                continue
            bw = usable
            if bw:
                rows = max(m - i0, 2 * bw)
                blk = fmat(rows, 2 * bw + 1, dev, fill=0.0)
                if me == owner:
                    blk[: m - i0, :bw] = Yp[:, :bw]
                    blk[:bw, bw:2 * bw] = T[:bw, :bw]
                    blk[:bw, 2 * bw] = tp[:bw]
                    blk[bw:2 * bw, bw:2 * bw] = P[:bw, :bw]        # R11
                    R[i0:i0 + bw, lp:lp + bw] = P[:bw, :bw]
                broadcast(blk, owner, group)
                Y[i0:, i0:i0 + bw] = blk[: m - i0, :bw]
                tau[i0:i0 + bw] = blk[:bw, 2 * bw]
                T = _f(blk[:bw, bw:2 * bw])
                R11 = _f(blk[bw:2 * bw, bw:2 * bw])
            break
        if bw == 0:
            rank_out = i0
            break
        nt2 = n - i0 - bw
        lc = layout.first_local_at_or_after(me, i0 + bw)
        if nt2:
            Yb = _f(Y[i0:, i0:i0 + bw])
            if work.shape[1] > lc:
                # G = Y_b^T A[i0:, mine] - (Y_b^T Y[i0:, :i0]) W[mine, :i0]^T   (truncated.py:144-149)
                G = K.gemm(Yb, _f(work[i0:, lc:]), transa=True)
                if i0:
                    Z = K.gemm(Yb, _f(Y[i0:, :i0]), transa=True)
                    K.gemm(Z, _f(Wt[:i0, lc:]), G, alpha=-1.0, beta=1.0)
                # W[mine, i0:i0+bw] = (T^T G)^T, stored transposed
                Wt[i0:i0 + bw, lc:] = K.gemm(T, G, transa=True)
                # R[i0:i0+bw, mine] = A[i0:i0+bw, mine] - Y[i0:i0+bw, :i0+bw] W[mine, :i0+bw]^T
                Rn = _f(work[i0:i0 + bw, lc:])
                K.gemm(_f(Y[i0:i0 + bw, :i0 + bw]), _f(Wt[:i0 + bw, lc:]), Rn, alpha=-1.0,
                       beta=1.0)
                R[i0:i0 + bw, lc:] = Rn
            ctr["gemm_flops"] += (2 * (m - i0) * bw * nt2
                                  + (2 * (m - i0) * bw * i0 + 2 * bw * i0 * nt2 if i0 else 0)
                                  + bw * bw * nt2 + 2 * bw * (i0 + bw) * nt2)
        i0 += bw
        if bw < want:
            rank_out = i0
            break
        if i0 < k:
            R12 = allgather_positions(_f(R[i0 - bw:i0, lc:]), layout, i0, me, group)
            Bn, degenerate = K.sample_update(S, bw, R11, _f(R12), frob)
            if degenerate:
                B = sketch(i0)
                ctr["resamples"] += 1
            else:
                B = Bn
                ctr["gemm_flops"] += 3 * bw * bw * (n - i0)
    R_local = R[:rank_out, :].clone()
    Wt_local = Wt[:rank_out, :].clone()
    Rg = Wg = None
    if gather:
        Rg = _f(allgather_positions(R_local, layout, 0, me, group))
        Wg = allgather_positions(Wt_local, layout, 0, me, group).t()
    return ShardedTruncated(Y=Y[:, :rank_out], tau=tau[:rank_out], perm=perm, swaps=swaps,
                            rank=rank_out, R_local=R_local, Wt_local=Wt_local, R=Rg, W=Wg,
                            layout=layout, counters=ctr)


def _f(t: torch.Tensor) -> torch.Tensor:
    """Column-major copy (or view) of a 2-D tensor for the C-ABI."""
    from .device import fmat, is_fortran
    if is_fortran(t):
        return t
    out = fmat(t.shape[0], t.shape[1], t.device)
    out.copy_(t)
    return out
