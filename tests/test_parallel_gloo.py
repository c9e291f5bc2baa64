"""Multi-rank host logic of the column-block-cyclic driver on CPU (gloo,
world_size 2): layout maps, the swap plan, the cross-rank column exchange and
the position-ordered all-gather -- checked against a single-process numpy
replay of the reference's swap semantics (randomized.py:138-147)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1509_06820_b200.parallel import (
    BlockCyclic,
    allgather_positions,
    exchange_columns,
    shard,
    swap_plan,
)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_layout_maps_are_a_bijection():
    for n, b, w in ((37, 4, 3), (64, 8, 2), (10, 16, 4), (1000, 32, 8)):
        L = BlockCyclic(n, b, w)
        seen = {}
        for r in range(w):
            for li, j in enumerate(L.positions(r)):
                assert L.owner(j) == r and L.local_index(j) == li
                seen[j] = (r, li)
        assert sorted(seen) == list(range(n))
        for r in range(w):
            p = L.positions(r)
            for pos in (0, b, n // 2, n - 1):
                lc = L.first_local_at_or_after(r, pos)
                assert np.all(p[lc:] >= pos) and np.all(p[:lc] < pos)


def _replay(A, piv, i0):
    A = A.copy()
    for j, p in enumerate(piv):
        a, c = i0 + j, i0 + p
        if a != c:
            A[:, [a, c]] = A[:, [c, a]]
    return A


def test_swap_plan_equals_sequential_swaps():
    g = np.random.default_rng(0)
    for trial in range(50):
        n = int(g.integers(8, 60))
        i0 = int(g.integers(0, n // 2))
        got = int(g.integers(1, min(8, n - i0) + 1))
        piv = [int(g.integers(j, n - i0)) for j in range(got)]
        A = g.standard_normal((3, n))
        ref = _replay(A, piv, i0)
        out = A.copy()
        moves = swap_plan(piv, got, i0)
        src = {d: A[:, s].copy() for d, s in moves}
        for d, col in src.items():
            out[:, d] = col
        np.testing.assert_array_equal(out, ref)


def _worker(rank, world, port, n, b, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.random.default_rng(seed)
        A = g.standard_normal((5, n))
        L = BlockCyclic(n, b, world)
        local = torch.from_numpy(shard(A, L, rank).copy())
        results = {}
        # a few rounds of block pivots, like the driver's per-block exchange
        full = A.copy()
        for i0 in range(0, n - b, b):
            got = b
            piv = [int(g.integers(j, n - i0)) for j in range(got)]
            full = _replay(full, piv, i0)
            exchange_columns(local, L, swap_plan(piv, got, i0), rank, None)
        results["local_ok"] = bool(np.array_equal(local.numpy(), shard(full, L, rank)))
        # position-ordered all-gather of the tail
        for pos0 in (0, b, n // 2):
            lc = L.first_local_at_or_after(rank, pos0)
            tail = allgather_positions(local[:, lc:], L, pos0, rank, None)
            results[f"gather_{pos0}"] = bool(np.array_equal(tail.numpy(), full[:, pos0:]))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,b", [(48, 4), (70, 8), (33, 16)])
def test_exchange_and_gather_world2(n, b):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, b, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out:
        assert all(res.values()), (rank, res)


# ---------------------------------------------------------------- the whole driver at world 2 / 3

def _driver_worker(rank, world, port_, kind, m, n, b, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_06820_b200.parallel import rqrcp_sharded
        from paper_1509_06820_b200.randomized import RandomizedConfig
        from tests import _cpu_kernels
        A = _driver_matrix(kind, m, n)
        L = BlockCyclic(n, b, world)
        local = torch.from_numpy(shard(A, L, rank).copy())
        f = rqrcp_sharded(local, m, n, None, RandomizedConfig(block=b, padding=8, seed=0),
                          gather_r=True, kernels=_cpu_kernels)
        q.put((rank, f.rank, f.perm.tolist(), f.swaps, f.R.numpy(), f.Y.numpy(),
               dict(f.counters)))
    finally:
        dist.destroy_process_group()


def _driver_matrix(kind, m, n):
    g = np.random.default_rng(11)
    if kind == "gauss":
        return g.standard_normal((m, n))
    if kind == "geom":   # 14 decades: resamples near the noise floor
        U = np.linalg.qr(g.standard_normal((m, m)))[0][:, :n]
        V = np.linalg.qr(g.standard_normal((n, n)))[0]
        return (U * 10.0 ** (-14.0 * np.arange(n) / (n - 1))) @ V.T
    return g.standard_normal((m, 9)) @ g.standard_normal((9, n))   # rank 9


@pytest.mark.parametrize("world,kind,m,n,b", [(2, "gauss", 60, 50, 8), (3, "gauss", 70, 64, 6),
                                              (2, "geom", 96, 80, 8), (3, "lowrank", 48, 40, 4)])
def test_sharded_driver_matches_single_process_reference(world, kind, m, n, b):
    """parallel.rqrcp_sharded runs its whole multi-rank control flow (sketch
    all-gather, replicated selection, cross-rank swaps, owner panel +
    broadcast, local trailing updates, R12 all-gather, sample update and
    resamples) on `world` gloo ranks, with oracle-backed kernels; the result
    must be the reference algorithm's (oracle/port.py = reference,
    tests/test_oracle_golden.py): same rank, pivots, swaps and resample
    count, R and Y to rounding -- up to the noise floor for rank-deficient
    inputs."""
    from oracle import port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_driver_worker, args=(r, world, port_, kind, m, n, b, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = _driver_matrix(kind, m, n)
    o = port.rqrcp(A, None, b, 8, 0)
    frob = np.linalg.norm(A)
    d = np.abs(np.diag(o.R))
    bad = d <= 1e3 * np.finfo(float).eps * frob
    r_sig = int(np.argmax(bad)) if bad.any() else d.size
    for rank, f_rank, perm, swaps, R, Y, ctr in out:
        # every rank holds the same replicated decisions
        assert perm == out[0][2] and swaps == out[0][3]
        np.testing.assert_array_equal(np.asarray(perm)[:r_sig], o.perm.forward[:r_sig])
        mine = np.zeros((R.shape[0], n))
        mine[:, perm] = R
        theirs = o.perm.restore(o.R)
        assert np.linalg.norm(mine[:r_sig] - theirs[:r_sig]) <= 1e-12 * np.linalg.norm(theirs[:r_sig])
        if r_sig == min(m, n):
            assert f_rank == o.rank
            assert swaps == [tuple(s) for s in o.perm.swaps]
            assert ctr["resamples"] == o.counters.resamples
            assert (ctr["gemm_flops"], ctr["level2_flops"]) == (o.counters.gemm_flops,
                                                               o.counters.level2_flops)
            assert np.linalg.norm(Y - o.Y) <= 1e-12 * np.linalg.norm(o.Y)


def _trq_worker(rank, world, port_, kind, m, n, k, b, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1509_06820_b200.parallel import trqrcp_sharded
        from paper_1509_06820_b200.randomized import RandomizedConfig
        from tests import _cpu_kernels
        A = _driver_matrix(kind, m, n)
        L = BlockCyclic(n, b, world)
        local = torch.from_numpy(shard(A, L, rank).copy())
        f = trqrcp_sharded(local, m, n, k, RandomizedConfig(block=b, padding=8, seed=0),
                           kernels=_cpu_kernels)
        q.put((rank, f.rank, f.perm.tolist(), f.swaps, f.R.numpy(), f.W.numpy(), f.Y.numpy(),
               dict(f.counters)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,m,n,k,b", [(2, "gauss", 60, 70, 32, 8),
                                                (3, "gauss", 64, 50, 30, 6),
                                                (2, "geom", 96, 80, 64, 8),
                                                (3, "lowrank", 48, 40, 20, 4)])
def test_sharded_trqrcp_matches_single_process_reference(world, kind, m, n, k, b):
    """parallel.trqrcp_sharded (truncated.py:70-174 control flow, A never
    updated, W rows and R columns following A's columns across ranks, the
    implicit resketch all-gathered) against the reference algorithm."""
    from oracle import port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_trq_worker, args=(r, world, port_, kind, m, n, k, b, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = _driver_matrix(kind, m, n)
    o = port.trqrcp(A, k, b, 8, 0)
    frob = np.linalg.norm(A)
    d = np.abs(np.diag(o.R))
    bad = d <= 1e3 * np.finfo(float).eps * frob
    r_sig = int(np.argmax(bad)) if bad.any() else d.size
    for rank, f_rank, perm, swaps, R, W, Y, ctr in out:
        assert perm == out[0][2] and swaps == out[0][3]
        np.testing.assert_array_equal(np.asarray(perm)[:r_sig], o.perm.forward[:r_sig])
        mine = np.zeros((R.shape[0], n))
        mine[:, perm] = R
        theirs = o.perm.restore(o.R)
        assert np.linalg.norm(mine[:r_sig] - theirs[:r_sig]) <= 1e-12 * np.linalg.norm(theirs[:r_sig])
        if r_sig == min(k, o.rank) and o.rank == k:
            assert f_rank == o.rank
            assert swaps == [tuple(s) for s in o.perm.swaps]
            assert ctr["resamples"] == o.counters.resamples
            assert (ctr["gemm_flops"], ctr["level2_flops"]) == (o.counters.gemm_flops,
                                                               o.counters.level2_flops)
            # a reflector (and W column) is determined to ~ eps ||A|| / |R_jj|
            # relative: compare column by column against that conditioning
            eps = np.finfo(float).eps
            for j in range(o.rank):
                tol_j = max(1e-12, 100 * eps * frob / d[j])
                assert np.linalg.norm(Y[:, j] - o.Y[:, j]) <= tol_j * np.linalg.norm(o.Y[:, j])
                assert np.linalg.norm(W[:, j] - o.W[:, j]) <= tol_j * max(np.linalg.norm(o.W[:, j]), 1e-300)
