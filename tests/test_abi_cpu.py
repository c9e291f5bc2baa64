"""CPU-only checks of the boundary: the C-ABI library loads without a GPU,
exports and types every symbol include/rqrcp_b200.h declares, and the host
side (argument validation, Omega stream, permutation semantics) behaves like
the reference.  No compute calls are made here."""

import os
import re

import numpy as np
import pytest

from tests import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rqrcp_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rq_[a-z0-9_]+)\s*\(", src)) - {"rq_omega_fn"})


def test_header_declares_entry_points():
    names = _declared()
    for must in ("rq_factor", "rq_tuxv", "rq_select_pivots", "rq_panel_qr", "rq_sample_update",
                 "rq_sketch", "rq_gemm", "rq_qr_blocked", "rq_q_columns", "rq_t_factor"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1509_06820_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        from paper_1509_06820_b200 import build
        build.build()
    lib = _abi.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _abi.SIGNATURES, f"{name} not typed in _abi.SIGNATURES"
    assert lib.rq_version() >= 100
    assert lib.rq_launch_count() >= 0


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_1509_06820_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.rqrcp(np.random.default_rng(0).standard_normal((20, 10)), 5,
                P.RandomizedConfig(block=4, padding=2))


def test_validation_messages_match_reference():
    """randomized.py:187-190, qrcp.py:91-93, truncated.py:220-221 -- raised
    before any device work."""
    import paper_1509_06820_b200 as P
    with pytest.raises(ValueError, match=r"rank 7 outside \[0, 6\]"):
        P.rqrcp(np.eye(6), 7)
    with pytest.raises(ValueError, match="rank must be >= 1"):
        P.rqrcp(np.eye(6), 0, P.RandomizedConfig(block=2, padding=2))
    with pytest.raises(ValueError, match="sample rows 10 exceed matrix rows 4"):
        P.ssrqrcp(np.diag([4.0, 3.0, 2.0, 1.0]), 2, P.RandomizedConfig(padding=8))
    with pytest.raises(ValueError, match="rank must be >= 1"):
        P.trqrcp(np.eye(6), 0, P.RandomizedConfig(block=2, padding=2))
    with pytest.raises(ValueError, match="j_max must be >= 1"):
        P.tuxv(np.eye(4), 2, P.RandomizedConfig(block=2, padding=2), j_max=0)
    with pytest.raises(ValueError, match="block must be >= 1"):
        P.RandomizedConfig(block=0)
    with pytest.raises(ValueError, match="padding must be >= 1"):
        P.RandomizedConfig(padding=0)
    assert P.RandomizedConfig(block=16, padding=8).ell == 24


def test_host_omega_stream_matches_reference_kats():
    import paper_1509_06820_b200 as P
    rec = G.load("kat_rng")
    st = P.RngState(0)
    np.testing.assert_array_equal(P.gaussian_matrix(st, 40, 8), rec["om40"])
    assert st.position == 320
    np.testing.assert_array_equal(P.gaussian_matrix(P.RngState(0, position=320), 40, 3),
                                  rec["tail"])
    buf = np.empty(72 * 2)
    P.RngState(0).fill(buf)
    np.testing.assert_array_equal(buf.reshape((72, 2), order="F"), rec["om72"])


def test_permutation_semantics():
    import paper_1509_06820_b200 as P
    p = P.Permutation.identity(5)
    for i, j in ((0, 3), (1, 1), (2, 4)):
        p.swap(i, j)
    assert list(p.forward) == [3, 1, 4, 0, 2]
    assert p.swaps == [(0, 3), (1, 1), (2, 4)]
    R = np.arange(10.0).reshape(2, 5)
    np.testing.assert_array_equal(p.restore(R)[:, p.forward], R)
    q = P.Permutation.from_order([3, 1, 4, 0, 2])
    assert list(q.forward) == [3, 1, 4, 0, 2]


def test_ssrqrcp_sample_beyond_the_pivot_kernel_rejected_before_any_device_work():
    import paper_1509_06820_b200 as P
    with pytest.raises(NotImplementedError, match="k = 4100"):
        P.ssrqrcp(np.zeros((4200, 4200)), 4100, P.RandomizedConfig(padding=8))
