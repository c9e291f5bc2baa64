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
