"""Kernel-level parity on the B200: each C-ABI primitive against the reference
fixtures (tests/golden/kat_*.npz) and the CPU oracle (oracle/port.py)."""

import numpy as np
import pytest

from oracle import port
from tests import _golden as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x):
    import paper_1509_06820_b200.device as D
    return D.to_device_fortran(x, torch.device("cuda", 0))


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", [(64, 96, 40), (130, 70, 3000), (7, 5, 3), (300, 257, 129),
                                   (72, 1000, 8192), (138, 202, 1030), (64, 100, 20000),
                                   (2050, 66, 48)])
def test_gemm_matches_fp64_reference(ta, tb, shape):
    from paper_1509_06820_b200.primitives import gemm
    m, n, k = shape
    g = np.random.default_rng(m * 7 + n + k)
    A = g.standard_normal((k, m) if ta else (m, k))
    B = g.standard_normal((n, k) if tb else (k, n))
    C0 = g.standard_normal((m, n))
    ref = (A.T if ta else A) @ (B.T if tb else B)
    for alpha, beta, want in ((1.0, 0.0, ref), (-1.0, 1.0, C0 - ref), (0.5, 2.0, 0.5 * ref + 2 * C0)):
        out = gemm(_dev(A), _dev(B), _dev(C0), alpha=alpha, beta=beta, transa=ta, transb=tb)
        got = out.cpu().numpy()
        # fp64 accumulation: error <= a few eps * k * |A||B|
        tol = 8 * k * np.finfo(float).eps * (np.abs(A).max() * np.abs(B).max() + np.abs(C0).max())
        assert np.max(np.abs(got - want)) <= tol, (alpha, beta)


def test_gemm_k_zero_scales_c():
    from paper_1509_06820_b200.primitives import gemm
    C0 = np.random.default_rng(0).standard_normal((10, 12))
    out = gemm(_dev(np.zeros((10, 0))), _dev(np.zeros((0, 12))), _dev(C0), alpha=1.0, beta=2.0)
    np.testing.assert_array_equal(out.cpu().numpy(), 2 * C0)


def test_select_pivots_matches_reference_fixtures():
    from paper_1509_06820_b200.primitives import select_pivots
    rec = G.load("kat_select")
    keys = sorted({k.rsplit("_", 1)[0] for k in rec})
    for key in keys:
        B = rec[f"{key}_B"]
        want = int(rec[f"{key}_want"])
        S, piv, got, Ys, taus, l2 = select_pivots(_dev(B), want)
        assert got == int(rec[f"{key}_got"]), key
        # replay the local swaps -> Permutation.forward
        fwd = list(range(B.shape[1]))
        for j, p in enumerate(piv):
            fwd[j], fwd[p] = fwd[p], fwd[j]
        np.testing.assert_array_equal(fwd, rec[f"{key}_perm"], err_msg=key)
        np.testing.assert_array_equal(np.array([(j, p) for j, p in enumerate(piv)]).reshape(-1, 2),
                                      rec[f"{key}_swaps"], err_msg=key)
        scale = float(np.linalg.norm(B))
        assert np.linalg.norm(S.cpu().numpy() - rec[f"{key}_S"]) <= 1e-12 * scale, key
        # tau of a rounding-noise column is arbitrary in [1, 2]; compare where |beta| is significant
        sig = np.abs(np.diag(rec[f"{key}_S"])[:got]) > 1e-8 * scale
        np.testing.assert_allclose(taus.cpu().numpy()[sig], rec[f"{key}_taus"][sig], rtol=1e-12, atol=1e-14)
        assert l2 == int(rec[f"{key}_l2"]), key
    assert list(rec["diag_perm"][:4]) == [1, 3, 0, 2]


def test_select_pivots_wide_sample_vs_oracle():
    from paper_1509_06820_b200.primitives import select_pivots
    g = np.random.default_rng(5)
    for ell, nt, want in ((72, 8192, 64), (40, 1000, 32), (136, 5000, 128), (20, 33, 12),
                          (300, 2000, 250), (264, 700, 256), (1100, 1500, 1050)):
        B = g.standard_normal((ell, nt)) * np.exp(g.uniform(-2, 2, nt))
        smp = port.Sample(B=np.asfortranarray(B.copy()), ell=ell)
        perm, got = port.pick_pivots(smp, want, port.Counters())
        S, piv, got_d, *_ = select_pivots(_dev(B), want)
        assert got_d == got
        fwd = list(range(nt))
        for j, p in enumerate(piv):
            fwd[j], fwd[p] = fwd[p], fwd[j]
        np.testing.assert_array_equal(fwd, perm.forward)
        assert np.linalg.norm(S.cpu().numpy() - smp.B) <= 1e-12 * np.linalg.norm(B)


def test_select_pivots_sample_wider_than_16_bit_positions():
    """nt > 65535: the argmax key switches to 20 position bits."""
    from paper_1509_06820_b200.primitives import select_pivots
    g = np.random.default_rng(70000)
    ell, nt, want = 40, 70000, 32
    B = g.standard_normal((ell, nt)) * np.exp(g.uniform(-2, 2, nt))
    # the largest columns at both ends of the position range
    B[:, 69999] *= 40.0
    B[:, 65536] *= 30.0
    B[:, 3] *= 20.0
    smp = port.Sample(B=np.asfortranarray(B.copy()), ell=ell)
    perm, got = port.pick_pivots(smp, want, port.Counters())
    S, piv, got_d, *_ = select_pivots(_dev(B), want)
    assert got_d == got
    assert max(int(p) for p in piv) > 65535   # a pivot beyond the 16-bit range
    fwd = list(range(nt))
    for j, p in enumerate(piv):
        fwd[j], fwd[p] = fwd[p], fwd[j]
    np.testing.assert_array_equal(fwd, perm.forward)
    assert np.linalg.norm(S.cpu().numpy() - smp.B) <= 1e-12 * np.linalg.norm(B)


@pytest.mark.parametrize("ell,nt,want,ctas", [(136, 5000, 128, 4), (72, 6000, 64, 3),
                                                (40, 3000, 32, 2), (160, 2500, 100, 2)])
def test_select_pivots_spilled_columns_vs_oracle(ell, nt, want, ctas):
    """The shared-memory selection kernel with most columns spilled to global
    memory (a few CTAs for a wide sample, as beside cfg5's trailing update):
    bit-for-bit the oracle's pivots, S to rounding, the same result as the
    register-resident path."""
    from paper_1509_06820_b200 import _abi
    from paper_1509_06820_b200.primitives import select_pivots
    lib, h = _abi.load_library(), _abi.handle(0)
    g = np.random.default_rng(ell + nt)
    B = g.standard_normal((ell, nt)) * np.exp(g.uniform(-2, 2, nt))
    smp = port.Sample(B=np.asfortranarray(B.copy()), ell=ell)
    perm, got = port.pick_pivots(smp, want, port.Counters())
    try:
        lib.rq_set_option(h, b"select_reg", 0)
        lib.rq_set_option(h, b"force_select", 1)
        lib.rq_set_option(h, b"select_max_ctas", ctas)
        S, piv, got_d, *_ = select_pivots(_dev(B), want)
    finally:
        lib.rq_set_option(h, b"select_reg", 1)
        lib.rq_set_option(h, b"force_select", 0)
        lib.rq_set_option(h, b"select_max_ctas", 0)
    assert got_d == got
    fwd = list(range(nt))
    for j, p in enumerate(piv):
        fwd[j], fwd[p] = fwd[p], fwd[j]
    np.testing.assert_array_equal(fwd, perm.forward)
    assert np.linalg.norm(S.cpu().numpy() - smp.B) <= 1e-12 * np.linalg.norm(B)


@pytest.mark.parametrize("ell,nt,want,ctas", [(72, 8128, 64, 44), (72, 3000, 64, 80), (40, 2000, 32, 0),
                                                (136, 3000, 128, 60), (72, 500, 64, 80)])
def test_select_fused_exchange_is_bitwise_the_barrier_variant(ell, nt, want, ctas):
    """Grid variant of the register-resident select: the fused exchange
    (barrier counter and key slot in one 16-byte word, one .b128 acquire poll)
    against the separate barrier + key read -- same pivots, S bit for bit, and
    stable over repeated launches (the {count, key} pairs are reset per
    launch); both equal the oracle's pivots."""
    from paper_1509_06820_b200 import _abi
    from paper_1509_06820_b200.primitives import select_pivots
    lib, h = _abi.load_library(), _abi.handle(0)
    g = np.random.default_rng(ell * nt)
    B = g.standard_normal((ell, nt)) * np.exp(g.uniform(-2, 2, nt))
    smp = port.Sample(B=np.asfortranarray(B.copy()), ell=ell)
    perm, got = port.pick_pivots(smp, want, port.Counters())
    out = {}
    try:
        lib.rq_set_option(h, b"force_select", 1)
        lib.rq_set_option(h, b"select_max_ctas", ctas)
        for fused in (1, 0, 1):
            lib.rq_set_option(h, b"select_fused", fused)
            S, piv, got_d, *_ = select_pivots(_dev(B), want)
            assert got_d == got
            out.setdefault(fused, []).append((S.cpu().numpy(), list(piv)))
    finally:
        lib.rq_set_option(h, b"select_fused", 1)
        lib.rq_set_option(h, b"force_select", 0)
        lib.rq_set_option(h, b"select_max_ctas", 0)
    S0, piv0 = out[0][0]
    for S1, piv1 in out[1]:
        assert piv1 == piv0
        np.testing.assert_array_equal(S1, S0)
    fwd = list(range(nt))
    for j, p in enumerate(piv0):
        fwd[j], fwd[p] = fwd[p], fwd[j]
    np.testing.assert_array_equal(fwd, perm.forward)


def test_panel_matches_reference_fixtures():
    from paper_1509_06820_b200.primitives import panel_qr
    rec = G.load("kat_panel")
    s = 0
    while f"p{s}_P" in rec:
        P = _dev(rec[f"p{s}_P"])
        Y, tau, T, usable, l2 = panel_qr(P)
        sc = float(np.linalg.norm(rec[f"p{s}_P"]))
        assert np.linalg.norm(P.cpu().numpy() - rec[f"p{s}_R"]) <= 1e-13 * sc
        assert np.linalg.norm(Y.cpu().numpy() - rec[f"p{s}_Y"]) <= 1e-12 * np.linalg.norm(rec[f"p{s}_Y"])
        np.testing.assert_allclose(tau.cpu().numpy(), rec[f"p{s}_tau"], rtol=1e-12, atol=1e-15)
        assert np.linalg.norm(T.cpu().numpy() - rec[f"p{s}_T"]) <= 1e-12 * np.linalg.norm(rec[f"p{s}_T"])
        assert l2 == int(rec[f"p{s}_l2"])
        assert usable == P.shape[1]
        s += 1


# (130, 64), (100, 20), (200, 33): fewer row chunks than the three CTAs the fast
# panel spreads its second serial section over (the grid is padded to 3)
@pytest.mark.parametrize("mm,bw", [(8192, 64), (32768, 128), (1000, 32), (257, 17), (130, 64),
                                   (100, 20), (200, 33)])
def test_panel_large_vs_oracle(mm, bw):
    from paper_1509_06820_b200.primitives import panel_qr
    P0 = np.random.default_rng(mm + bw).standard_normal((mm, bw))
    Pc = np.asfortranarray(P0.copy())
    Yo, to = port.panel_qr(Pc)
    P = _dev(P0)
    Y, tau, T, usable, _ = panel_qr(P)
    assert np.linalg.norm(P.cpu().numpy() - Pc) <= 1e-13 * np.linalg.norm(P0)
    assert np.linalg.norm(Y.cpu().numpy() - Yo) <= 1e-12 * np.linalg.norm(Yo)
    np.testing.assert_allclose(T.cpu().numpy(), port.t_factor(Yo, to), rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("b", [64, 128])
def test_sample_update_vs_oracle(b):
    from paper_1509_06820_b200.primitives import sample_update
    g = np.random.default_rng(3)
    ell, nt = b + 8, 700
    B = g.standard_normal((ell, nt))
    smp = port.Sample(B=np.asfortranarray(B.copy()), ell=ell, frob_a=10.0)
    port.pick_pivots(smp, b, port.Counters())
    S = smp.B.copy()
    R11 = np.triu(g.standard_normal((b, b))) + 4 * np.eye(b)
    R12 = g.standard_normal((b, nt - b))
    port.downdate_sample(smp, R11, R12, port.Counters())
    Bn, deg = sample_update(_dev(S), b, _dev(R11), _dev(R12), 10.0)
    assert not deg
    assert np.linalg.norm(Bn.cpu().numpy() - smp.B) <= 1e-11 * np.linalg.norm(smp.B)
    R11[5, 5] = 1e-300
    _, deg = sample_update(_dev(S), b, _dev(R11), _dev(R12), 10.0)
    assert deg


def _panel_with(P0, fast, **kw):
    from paper_1509_06820_b200 import _abi
    from paper_1509_06820_b200.primitives import panel_qr
    lib, h = _abi.load_library(), _abi.handle(0)
    lib.rq_set_option(h, b"fast_panel", int(fast))
    try:
        P = _dev(P0)
        Y, tau, T, usable, l2 = panel_qr(P, **kw)
        torch.cuda.synchronize()
        return (P.cpu().numpy(), Y.cpu().numpy(), tau.cpu().numpy(), T.cpu().numpy(), usable, l2)
    finally:
        lib.rq_set_option(h, b"fast_panel", 1)


@pytest.mark.parametrize("mm,bw", [(8192, 64), (4096, 64), (1000, 32), (130, 64), (20000, 32),
                                   (300, 16), (97, 8)])
def test_fast_panel_matches_oracle(mm, bw):
    """CholeskyQR2 + Householder reconstruction (panel_fast.cu) reproduces the
    reference's reflectors (beta = -sign(alpha)||x||) to rounding level."""
    P0 = np.random.default_rng(mm * 3 + bw).standard_normal((mm, bw))
    P0 *= np.logspace(0, -1.5, bw)[None, :]
    Pc = np.asfortranarray(P0.copy())
    Yo, to = port.panel_qr(Pc)
    R, Y, tau, T, usable, l2 = _panel_with(P0, True)
    Re, Ye, taue, Te, usable_e, l2e = _panel_with(P0, False)
    assert not np.array_equal(R, Re), "fast path did not run"
    assert np.linalg.norm(R - Pc) <= 1e-13 * np.linalg.norm(P0)
    assert np.linalg.norm(Y - Yo) <= 1e-12 * np.linalg.norm(Yo)
    np.testing.assert_allclose(tau, to, rtol=1e-13, atol=0)
    assert np.all((tau >= 1.0) & (tau <= 2.0))
    np.testing.assert_allclose(T, port.t_factor(Yo, to), rtol=1e-10, atol=1e-13)
    assert (usable, l2) == (usable_e, l2e) == (bw, l2)
    # the shared-memory row stride is a layout choice only: bitwise the same
    from paper_1509_06820_b200 import _abi
    lib, h = _abi.load_library(), _abi.handle(0)
    try:
        for pad in (1, 8):
            lib.rq_set_option(h, b"fast_panel_pad", pad)
            got = _panel_with(P0, True)
            for x, y in zip(got[:4], (R, Y, tau, T)):
                np.testing.assert_array_equal(x, y)
    finally:
        lib.rq_set_option(h, b"fast_panel_pad", 4)


@pytest.mark.parametrize("kind", ["dup", "tiny_col", "zero_col", "near_tol"])
def test_fast_panel_declines_to_exact_kernel(kind):
    """Rank-deficient / ill-conditioned / near-threshold panels fall back to the
    column-by-column kernel: results are bitwise those of the exact path."""
    mm, bw = 2048, 64
    P0 = np.random.default_rng(5).standard_normal((mm, bw))
    kw = {}
    if kind == "dup":
        P0[:, 40] = P0[:, 3]
    elif kind == "tiny_col":
        P0[:, -1] *= 1e-8
    elif kind == "zero_col":
        P0[:, 7] = 0.0
    else:   # a column whose R diagonal sits just above the usable threshold
        P0[:, -1] *= 1e-12
        kw["tol"] = 1e-13 * np.linalg.norm(P0[:, -1])
    a = _panel_with(P0, True, **kw)
    b = _panel_with(P0, False, **kw)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)
    assert a[4:] == b[4:]


@pytest.mark.parametrize("nb", [1, 7, 32, 40, 64])
def test_t_factor_inverse_matches_recurrence(nb):
    """T as the DMMA inverse of striu(Y^T Y) + diag(1/tau) against the
    reference recurrence (kernels.py:139-147), with tau = 0 (identity)
    reflectors mixed in."""
    from paper_1509_06820_b200 import _abi
    from paper_1509_06820_b200.factorization import t_factor
    g = np.random.default_rng(nb)
    mm = 300
    Y = np.tril(g.standard_normal((mm, nb)), -1)
    Y[np.arange(nb), np.arange(nb)] = 1.0
    tau = 2.0 / np.sum(Y * Y, axis=0)
    if nb > 3:
        tau[[1, nb - 2]] = 0.0
    lib, h = _abi.load_library(), _abi.handle(0)
    ref = port.t_factor(Y, tau)
    got = t_factor(Y, tau)
    lib.rq_set_option(h, b"t_inverse", 0)
    try:
        rec = t_factor(Y, tau)
    finally:
        lib.rq_set_option(h, b"t_inverse", 1)
    scale = np.linalg.norm(ref)
    assert np.linalg.norm(got - ref) <= 1e-13 * scale
    assert np.linalg.norm(rec - ref) <= 1e-13 * scale
    np.testing.assert_array_equal(got[np.tril_indices(nb, -1)], 0.0)


@pytest.mark.parametrize("M,N,K", [(20000, 224, 32), (5000, 1000, 32), (20000, 224, 64),
                                   (4100, 3000, 64), (8192, 256, 128), (300, 100, 32),
                                   (4100, 3002, 128), (130, 70, 64), (66, 2, 32)])
def test_rank_update_multi_tile(M, N, K):
    """C -= Y X through the persistent rank-b kernels when a CTA owns several
    tiles (tall trailing blocks; K = 128 as two 64-deep passes), against
    the fp64 numpy product."""
    from paper_1509_06820_b200.primitives import gemm
    g = np.random.default_rng(M + N + K)
    Y, X, C0 = g.standard_normal((M, K)), g.standard_normal((K, N)), g.standard_normal((M, N))
    out = gemm(_dev(Y), _dev(X), _dev(C0), alpha=-1.0, beta=1.0).cpu().numpy()
    assert np.abs(out - (C0 - Y @ X)).max() <= 64 * K * np.finfo(float).eps * 10
    # the grouped TMA kernel's variants (C from HBM; C tile prefetched by TMA
    # with k 16 / k 8 stages) run the same DMMA order: bitwise identical
    from paper_1509_06820_b200 import _abi
    lib, h = _abi.load_library(), _abi.handle(0)
    try:
        for v in (1, 3):
            lib.rq_set_option(h, b"ru_tma", v)
            alt = gemm(_dev(Y), _dev(X), _dev(C0), alpha=-1.0, beta=1.0).cpu().numpy()
            np.testing.assert_array_equal(alt, out)
    finally:
        lib.rq_set_option(h, b"ru_tma", 2)
