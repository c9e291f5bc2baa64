"""Pin the CPU oracle (oracle/port.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
(/root/reference/pkg/src/rqrcp) in the build container; see
tests/golden/make_golden.py.  On the CPU that generated them the oracle is
bitwise identical; elsewhere (different OpenBLAS kernels) the pivots must
still be identical and floats agree to rounding level.
"""

import numpy as np
import pytest

from oracle import port
from tests import _golden as G

EPS = np.finfo(np.float64).eps


def _run_oracle(rec, A):
    drv = str(rec["driver"])
    args = (A, G.k_of(rec), int(rec["block"]), int(rec["padding"]), int(rec["seed"]))
    if drv == "tuxv":
        return port.tuxv(*args)
    return getattr(port, drv)(*args)


def _close(a, b, scale, rel=1e-12):
    assert a.shape == b.shape
    assert np.linalg.norm(a - b) <= rel * max(scale, 1e-300)


@pytest.mark.parametrize("name", G.case_names())
def test_oracle_matches_reference_fixture(name):
    rec = G.load(name)
    A = G.matrix_of(rec)
    f = _run_oracle(rec, A)
    frob = float(np.linalg.norm(A))
    assert f.rank == int(rec["rank"])
    if str(rec["driver"]) == "tuxv":
        _close(f.singular_values(), rec["sv"], frob)
        _close(f.approx(), rec["U"] @ (rec["X"] @ rec["V"].T), frob)
        assert f.counters.gemm_flops == int(rec["gemm_flops"])
        return
    c = f.counters
    assert (c.gemm_flops, c.level2_flops, c.bytes_touched, c.resamples) == (
        int(rec["gemm_flops"]), int(rec["level2_flops"]), int(rec["bytes_touched"]),
        int(rec["resamples"]))
    np.testing.assert_array_equal(f.perm.forward, rec["perm"])
    np.testing.assert_array_equal(np.asarray(f.perm.swaps, dtype=np.int64).reshape(-1, 2),
                                  rec["swaps"])
    if "R" in rec:
        _close(f.R, rec["R"], frob)
        _close(f.Y, rec["Y"], 1.0)
        _close(f.tau, rec["tau"], 1.0)
        if "W" in rec:
            _close(f.W, rec["W"], frob)
        if "trailing" in rec:
            _close(f.trailing, rec["trailing"], frob)
    else:
        np.testing.assert_allclose(np.diag(f.R), rec["R_diag"], rtol=1e-10, atol=1e-13 * frob)
        np.testing.assert_allclose(f.R[:8], rec["R_head"], rtol=0, atol=1e-12 * frob)
        _close(f.tau, rec["tau"], 1.0)


def test_oracle_bitwise_on_generating_host():
    """Same numpy calls in the same order: on the fixture host the oracle's
    config-1 R is bit-identical to the reference's (sha256 of the bytes)."""
    rec = G.load("cfg1_rq_gauss_1000")
    f = port.rqrcp(G.matrix_of(rec), None, 32, 8, 0)
    same = G.sha(f.R) == str(rec["sha_R"])
    if not same:
        pytest.skip("different BLAS build than the fixture host; tolerance test covers it")
    assert G.sha(f.Y) == str(rec["sha_Y"])


def test_rng_stream_kats():
    rec = G.load("kat_rng")
    s = port.Stream(0)
    np.testing.assert_array_equal(s.matrix(40, 8), rec["om40"])
    np.testing.assert_array_equal(s.matrix(40, 3), rec["tail"])
    np.testing.assert_array_equal(port.Stream(0, position=320).matrix(40, 3), rec["tail"])
    np.testing.assert_array_equal(port.Stream(0).matrix(72, 2), rec["om72"])
    # SURVEY.md Appendix B known answers
    assert rec["om40"][0, 0] == 0.15929546600623282
    assert rec["om40"][1, 0] == -1.7741885208017214


def test_reflector_kats():
    rec = G.load("kat_reflector")
    i = 0
    while f"x{i}" in rec:
        v, tau, beta = port.householder(rec[f"x{i}"])
        r = rec[f"r{i}"]
        assert tau == r[0] and beta == r[1]
        np.testing.assert_array_equal(v, r[2:])
        i += 1
    v, tau, beta = port.householder(np.array([3.0, 4.0]))
    assert beta == -5.0 and tau == 1.6 and list(v) == [1.0, 0.5]


def test_select_kats():
    rec = G.load("kat_select")
    keys = sorted({k.rsplit("_", 1)[0] for k in rec})
    for key in keys:
        B = np.asfortranarray(rec[f"{key}_B"].copy())
        smp = port.Sample(B=B, ell=B.shape[0])
        ctr = port.Counters()
        perm, got = port.pick_pivots(smp, int(rec[f"{key}_want"]), ctr)
        assert got == int(rec[f"{key}_got"]), key
        np.testing.assert_array_equal(perm.forward, rec[f"{key}_perm"])
        np.testing.assert_array_equal(np.asarray(perm.swaps).reshape(-1, 2), rec[f"{key}_swaps"])
        scale = float(np.linalg.norm(rec[f"{key}_B"]))
        _close(smp.B, rec[f"{key}_S"], scale)
        assert ctr.level2_flops == int(rec[f"{key}_l2"])
    assert list(rec["diag_perm"][:4]) == [1, 3, 0, 2]


def test_panel_kats():
    rec = G.load("kat_panel")
    s = 0
    while f"p{s}_P" in rec:
        P = np.asfortranarray(rec[f"p{s}_P"].copy())
        ctr = port.Counters()
        Y, tau = port.panel_qr(P, ctr)
        sc = float(np.linalg.norm(rec[f"p{s}_P"]))
        _close(P, rec[f"p{s}_R"], sc)
        _close(Y, rec[f"p{s}_Y"], float(np.linalg.norm(rec[f"p{s}_Y"])))
        _close(tau, rec[f"p{s}_tau"], 2.0)
        _close(port.t_factor(Y, tau), rec[f"p{s}_T"], float(np.linalg.norm(rec[f"p{s}_T"])))
        assert ctr.level2_flops == int(rec[f"p{s}_l2"])
        s += 1


def test_oracle_validation_errors():
    with pytest.raises(ValueError, match="rank"):
        port.rqrcp(np.eye(6), 7)
    with pytest.raises(ValueError, match="rank must be >= 1"):
        port.rqrcp(np.eye(6), 0, 2, 2)
    with pytest.raises(ValueError, match="sample rows"):
        port.ssrqrcp(np.diag([4.0, 3.0, 2.0, 1.0]), 2, padding=8)
    with pytest.raises(ValueError):
        port.tuxv(np.eye(4), 2, 2, 2, j_max=0)


def test_explicit_omega_equals_seeded_stream():
    A = np.random.default_rng(3).standard_normal((50, 40))
    om = port.Stream(4).matrix(12, 50)
    f1 = port.rqrcp(A, 24, 8, 4, 4)
    f2 = port.rqrcp(A, 24, 8, 4, 4, omega=om)
    np.testing.assert_array_equal(f1.perm.forward, f2.perm.forward)
    np.testing.assert_array_equal(f1.R, f2.R)


def test_qr_presorted_kats():
    """qr_blocked / qr_presorted / column_norms (qrcp.py:222-268,
    kernels.py:184-186): the oracle reproduces the reference's fixture bit for
    bit on the generating host (C-order, F-order, tied norms, partial rank)."""
    rec = G.load("kat_qr_presorted")
    for key in sorted({k.split("_")[0] for k in rec}):
        A = rec[f"{key}_A"]
        if int(rec[f"{key}_forder"]):
            A = np.asfortranarray(A)
        k = int(rec[f"{key}_k"])
        k = None if k < 0 else k
        b = int(rec[f"{key}_b"])
        np.testing.assert_array_equal(port.column_norms(A), rec[f"{key}_norms"])
        ctr = port.Counters()
        Y, tau, R, order = port.qr_presorted(A, k, b, ctr)
        np.testing.assert_array_equal(order, rec[f"{key}_perm"])
        np.testing.assert_array_equal(R, rec[f"{key}_R"])
        np.testing.assert_array_equal(tau, rec[f"{key}_tau"])
        assert [ctr.gemm_flops, ctr.level2_flops, ctr.bytes_touched] == list(rec[f"{key}_counters"])
        cb = port.Counters()
        _, _, Rb = port.qr_blocked(A, k, b, cb)
        np.testing.assert_array_equal(Rb, rec[f"{key}_blocked_R"])
        assert [cb.gemm_flops, cb.level2_flops, cb.bytes_touched] == list(rec[f"{key}_blocked_counters"])
