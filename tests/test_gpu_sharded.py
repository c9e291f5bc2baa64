"""The column-block-cyclic driver (paper_1509_06820_b200/parallel.py) on the
B200 with a single-rank NCCL group must reproduce the native single-GPU
driver: same pivots, same resamples, R to rounding.  The native driver runs
with the same G = Y^T C arithmetic as the sharded one (option overlap_inner
off): its default splits G through the fast panel's M, a different rounding
that near-tie fixtures (noise-floor pivots) are sensitive to; parity with the
reference itself is tested in test_gpu_drivers.py."""

import os
import socket

import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_1509_06820_b200 import _abi
    lib, h = _abi.load_library(), _abi.handle(0)
    lib.rq_set_option(h, b"overlap_inner", 0)
    yield None
    lib.rq_set_option(h, b"overlap_inner", 1)
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rq_gauss_130x97_full", "rq_geom16_128_b8", "rq_gauss_60x45_k20",
                                  "cfg1_rq_gauss_1000"])
def test_sharded_world1_matches_native(group, name):
    import torch
    import paper_1509_06820_b200 as P
    from paper_1509_06820_b200.parallel import rqrcp_sharded
    rec = G.load(name)
    A = G.matrix_of(rec)
    cfg = P.RandomizedConfig(block=int(rec["block"]), padding=int(rec["padding"]),
                             seed=int(rec["seed"]))
    f = P.rqrcp(A, G.k_of(rec), cfg)
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    s = rqrcp_sharded(Ad, A.shape[0], A.shape[1], G.k_of(rec), cfg)
    assert s.rank == f.rank
    np.testing.assert_array_equal(s.perm, np.asarray(f.perm.forward))
    assert s.counters["resamples"] == f.counters.resamples
    R = s.R.cpu().numpy()
    assert np.linalg.norm(R - f.R) <= 1e-12 * max(np.linalg.norm(f.R), 1e-300)
    np.testing.assert_array_equal(np.array(s.swaps).reshape(-1, 2),
                                  np.array(f.perm.swaps).reshape(-1, 2))


@pytest.mark.parametrize("m,n,b", [(2048, 1800, 64), (1500, 1500, 48), (1200, 1000, 128)])
def test_sharded_world1_larger_vs_oracle(group, m, n, b):
    """Larger and odd block widths through the sharded driver against the CPU
    oracle (pivots identical, R to 1e-10)."""
    import torch
    import paper_1509_06820_b200 as P
    from oracle import port
    from paper_1509_06820_b200.parallel import rqrcp_sharded
    A = np.random.default_rng(m + b).standard_normal((m, n))
    cfg = P.RandomizedConfig(block=b, padding=8, seed=0)
    o = port.rqrcp(A, None, b, 8, 0)
    s = rqrcp_sharded(torch.from_numpy(np.asfortranarray(A)).cuda(), m, n, None, cfg)
    np.testing.assert_array_equal(s.perm, o.perm.forward)
    assert np.linalg.norm(s.R.cpu().numpy() - o.R) <= 1e-10 * np.linalg.norm(o.R)


@pytest.mark.parametrize("m,n,k,b", [(1200, 1000, 256, 64), (2000, 1500, 300, 32)])
def test_sharded_trqrcp_world1_vs_oracle(group, m, n, k, b):
    """The column-block-cyclic TRQRCP driver (parallel.trqrcp_sharded) on the
    B200 through NCCL: pivots identical to the reference algorithm, R and W
    to 1e-10."""
    import torch
    import paper_1509_06820_b200 as P
    from oracle import port
    from paper_1509_06820_b200.parallel import trqrcp_sharded
    A = np.random.default_rng(m + k).standard_normal((m, n))
    cfg = P.RandomizedConfig(block=b, padding=8, seed=0)
    o = port.trqrcp(A, k, b, 8, 0)
    s = trqrcp_sharded(torch.from_numpy(np.asfortranarray(A)).cuda(), m, n, k, cfg)
    assert s.rank == o.rank
    np.testing.assert_array_equal(s.perm, o.perm.forward)
    assert np.linalg.norm(s.R.cpu().numpy() - o.R) <= 1e-10 * np.linalg.norm(o.R)
    assert np.linalg.norm(s.W.cpu().numpy() - o.W) <= 1e-10 * np.linalg.norm(o.W)
    assert s.counters["resamples"] == o.counters.resamples
