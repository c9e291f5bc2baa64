"""Driver-level parity on the B200: every reference-generated fixture
(tests/golden/*.npz) re-run through the drop-in API (C-ABI underneath).

Bars (BASELINE north_star): identical pivot permutation; R within 1e-10
relative; ||AP - QR||_F/||A||_F <= 1e-12; ||Q^T Q - I|| <= 1e-12; identical
OpCounters (gemm, level-2, bytes, resamples) and rank; TUXV singular values
and approximation within 1e-9 relative of the reference.
"""

import numpy as np
import pytest

from oracle import port
from tests import _golden as G

pytestmark = pytest.mark.gpu


def _cfg(rec):
    import paper_1509_06820_b200 as P
    return P.RandomizedConfig(block=int(rec["block"]), padding=int(rec["padding"]),
                              seed=int(rec["seed"]))


def _run(rec, A, **kw):
    import paper_1509_06820_b200 as P
    drv = str(rec["driver"])
    return getattr(P, drv)(A, G.k_of(rec), _cfg(rec), **kw)


EPS = np.finfo(np.float64).eps
NOISE = 1e3  # pivots with |R_jj| <= NOISE * eps * ||A||_F are decided by rounding noise


def noise_floor_rank(rec, frob):
    """Leading pivots of the reference that sit above the FP64 rounding floor.
    Past this index the reference itself is choosing among columns whose
    residual norms are O(eps ||A||): those decisions (pivot order, tau = 0
    skips, the rank cut-off) are near-ties within the rounding margin
    (north_star)."""
    d = np.abs(np.diag(rec["R"]) if "R" in rec else rec["R_diag"])
    bad = d <= NOISE * EPS * frob
    return int(np.argmax(bad)) if bad.any() else d.size


@pytest.mark.parametrize("name", G.case_names())
def test_driver_matches_reference_fixture(name):
    rec = G.load(name)
    A = G.matrix_of(rec)
    f = _run(rec, A)
    frob = float(np.linalg.norm(A))
    drv = str(rec["driver"])
    if drv == "tuxv":
        assert f.rank == int(rec["rank"])
        np.testing.assert_allclose(f.singular_values(), rec["sv"], rtol=1e-9, atol=1e-12 * frob)
        ref = rec["U"] @ (rec["X"] @ rec["V"].T)
        assert np.linalg.norm(f.approx() - ref) <= 1e-9 * frob
        assert f.counters.gemm_flops == int(rec["gemm_flops"])
        assert f.counters.level2_flops == int(rec["level2_flops"])
        return
    ref_rank = int(rec["rank"])
    k_req = G.k_of(rec) if G.k_of(rec) is not None else min(A.shape)
    r_sig = noise_floor_rank(rec, frob)
    strict = ref_rank == k_req and r_sig == ref_rank
    pf = np.asarray(f.perm.forward)
    if strict:
        # every decision above the noise floor: bitwise-identical control flow
        assert f.rank == ref_rank
        c = f.counters
        assert (c.gemm_flops, c.level2_flops, c.bytes_touched, c.resamples) == (
            int(rec["gemm_flops"]), int(rec["level2_flops"]), int(rec["bytes_touched"]),
            int(rec["resamples"]))
        np.testing.assert_array_equal(pf, rec["perm"])
        np.testing.assert_array_equal(np.array(f.perm.swaps, dtype=np.int64).reshape(-1, 2),
                                      rec["swaps"])
        if "R" in rec:
            assert np.linalg.norm(f.R - rec["R"]) <= 1e-10 * max(np.linalg.norm(rec["R"]), 1e-300)
            if "trailing" in rec and rec["trailing"].size:
                assert np.linalg.norm(f.trailing - rec["trailing"]) <= 1e-10 * frob
            if "W" in rec:
                assert np.linalg.norm(f.reflectors.W - rec["W"]) <= 1e-10 * frob
        else:
            np.testing.assert_allclose(np.diag(f.R), rec["R_diag"], rtol=1e-10, atol=1e-12 * frob)
    else:
        # identical pivots and R rows (original column frame) above the floor
        assert f.rank >= r_sig
        np.testing.assert_array_equal(pf[:r_sig], rec["perm"][:r_sig])
        if "R" in rec and r_sig:
            mine = f.perm.restore(f.R)[:r_sig]
            theirs = np.zeros_like(rec["R"])
            theirs[:, rec["perm"]] = rec["R"]
            assert np.linalg.norm(mine - theirs[:r_sig]) <= 1e-10 * np.linalg.norm(theirs[:r_sig])
    if f.rank:
        q = f.q_factor()
        assert np.linalg.norm(q.T @ q - np.eye(f.rank), 2) <= 1e-12
        if drv in ("rqrcp", "rsrqrcp"):
            rebuilt = np.zeros(A.shape)
            rebuilt[: f.rank] = f.R
            rebuilt[f.rank:, f.rank:] = f.trailing
            res = np.linalg.norm(A[:, f.perm.forward] - f.q_factor(full=True) @ rebuilt)
            assert res <= 1e-12 * frob


def test_explicit_omega_matches_seeded_stream():
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(3).standard_normal((200, 150))
    cfg = P.RandomizedConfig(block=16, padding=8, seed=4)
    om = P.gaussian_matrix(P.RngState(4), cfg.ell, 200)
    f1 = P.rqrcp(A, None, cfg)
    f2 = P.rqrcp(A, None, cfg, omega=om)
    np.testing.assert_array_equal(f1.perm.forward, f2.perm.forward)
    np.testing.assert_array_equal(f1.R, f2.R)


def test_deterministic_and_device_inputs():
    import torch
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(4).standard_normal((500, 400))
    cfg = P.RandomizedConfig(block=32, padding=8, seed=11)
    f1 = P.rqrcp(A, 256, cfg)
    f2 = P.rqrcp(A, 256, cfg)
    np.testing.assert_array_equal(f1.R, f2.R)
    fd = P.rqrcp(torch.from_numpy(A).cuda(), 256, cfg)
    assert fd.R.is_cuda
    np.testing.assert_array_equal(fd.R.cpu().numpy(), f1.R)


def test_validation_errors_match_reference():
    import paper_1509_06820_b200 as P
    with pytest.raises(ValueError, match="rank 7 outside"):
        P.rqrcp(np.eye(6), 7)
    with pytest.raises(ValueError, match="rank must be >= 1"):
        P.rqrcp(np.eye(6), 0, P.RandomizedConfig(block=2, padding=2))
    with pytest.raises(ValueError, match="sample rows"):
        P.ssrqrcp(np.diag([4.0, 3.0, 2.0, 1.0]), 2, P.RandomizedConfig(padding=8))
    with pytest.raises(ValueError, match="j_max"):
        P.tuxv(np.eye(4), 2, P.RandomizedConfig(block=2, padding=2), j_max=0)
    with pytest.raises(ValueError):
        P.RandomizedConfig(block=0)


@pytest.mark.parametrize("n,b", [(2048, 64), (1536, 128), (3072, 32)])
def test_rqrcp_larger_vs_oracle(n, b):
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(n).standard_normal((n, n))
    o = port.rqrcp(A, None, b, 8, 0)
    f = P.rqrcp(A, None, P.RandomizedConfig(block=b, padding=8, seed=0))
    np.testing.assert_array_equal(f.perm.forward, o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)
    assert f.counters.gemm_flops == o.counters.gemm_flops
    # b = 128: the panel runs as two fast 64-column halves; the level-2 count
    # still equals the reference's column-by-column panels
    assert f.counters.level2_flops == o.counters.level2_flops


def test_trqrcp_tuxv_vs_oracle_mid_size():
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(1)
    A = g.standard_normal((3000, 200)) @ g.standard_normal((200, 2500)) \
        + 1e-6 * g.standard_normal((3000, 2500))
    cfg = P.RandomizedConfig(block=32, padding=8, seed=0)
    o = port.trqrcp(A, 256, 32, 8, 0)
    f = P.trqrcp(A, 256, cfg)
    np.testing.assert_array_equal(f.perm.forward, o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)
    ot = port.tuxv(A, 128, 32, 8, 0)
    ft = P.tuxv(A, 128, cfg)
    np.testing.assert_allclose(ft.singular_values(), ot.singular_values(), rtol=1e-9)


def test_qr_blocked_presorted_vs_reference():
    """qr_blocked / qr_presorted / column_norms on the GPU (qrcp.py:222-268,
    kernels.py:184-186) against the reference's fixture: bit-identical column
    norms for the caller's layout (so tied norms sort identically), the same
    permutation and counters, R within 1e-10."""
    import paper_1509_06820_b200 as P
    rec = G.load("kat_qr_presorted")
    for key in sorted({k.split("_")[0] for k in rec}):
        A = rec[f"{key}_A"]
        if int(rec[f"{key}_forder"]):
            A = np.asfortranarray(A)
        k = int(rec[f"{key}_k"])
        k = None if k < 0 else k
        b = int(rec[f"{key}_b"])
        np.testing.assert_array_equal(P.column_norms(A), rec[f"{key}_norms"], err_msg=key)
        f = P.qr_presorted(A, k, b)
        np.testing.assert_array_equal(np.asarray(f.perm.forward), rec[f"{key}_perm"], err_msg=key)
        scale = np.linalg.norm(rec[f"{key}_R"])
        assert np.linalg.norm(f.R - rec[f"{key}_R"]) <= 1e-10 * scale, key
        assert np.linalg.norm(f.trailing - rec[f"{key}_trailing"]) <= 1e-10 * scale, key
        c = f.counters
        assert [c.gemm_flops, c.level2_flops, c.bytes_touched] == list(rec[f"{key}_counters"]), key
        fb = P.qr_blocked(A, k, b)
        assert np.linalg.norm(fb.R - rec[f"{key}_blocked_R"]) <= 1e-10 * scale, key
        cb = fb.counters
        assert [cb.gemm_flops, cb.level2_flops, cb.bytes_touched] == \
            list(rec[f"{key}_blocked_counters"]), key
        q = f.q_factor()
        Ap = A[:, f.perm.forward]
        assert np.linalg.norm(Ap[:, :f.rank] - q @ f.R[:, :f.rank]) <= 1e-12 * np.linalg.norm(A), key


def test_reference_plain_qr_small_cases():
    """Small known answers of the reference's plain-QR tests
    (tests/test_qrcp.py): identity, block-size invariance on 64 x 48, wide and
    tall 9 x 17 / 17 x 9 inputs with the full Q, presorted diag(1, 3, 2), ties
    kept in order, the first diagonal equal to the largest column norm."""
    import paper_1509_06820_b200 as P

    def rec_err(f, A):
        m, n = A.shape
        rebuilt = np.zeros((m, n))
        rebuilt[: f.rank] = f.R
        if f.trailing is not None:
            rebuilt[f.rank:, f.rank:] = f.trailing
        return np.linalg.norm(A[:, np.asarray(f.perm.forward)] - f.q_factor(full=True) @ rebuilt) / np.linalg.norm(A)

    np.testing.assert_allclose(np.abs(P.qr_blocked(np.eye(3)).R), np.eye(3))
    A = np.random.default_rng(8).standard_normal((64, 48))
    f1, f2 = P.qr_blocked(A, b=16), P.qr_blocked(A, b=48)
    np.testing.assert_allclose(f1.R, f2.R, atol=50 * EPS * 64 * np.linalg.norm(A))
    assert rec_err(f1, A) <= 100 * EPS * 64
    g = np.random.default_rng(10)
    for shape in ((9, 17), (17, 9)):
        A = g.standard_normal(shape)
        f = P.qr_blocked(A, b=4)
        o = port.qr_blocked(np.asfortranarray(A.copy()), b=4)
        assert np.linalg.norm(f.R - o[2][: f.R.shape[0]]) <= 1e-12 * np.linalg.norm(A)
        assert rec_err(f, A) <= 100 * EPS * max(shape)
        Q = f.q_factor(full=True)
        assert np.linalg.norm(Q.T @ Q - np.eye(shape[0])) <= 100 * EPS * max(shape)
    f = P.qr_presorted(np.diag([1.0, 3.0, 2.0]))
    assert list(f.perm.forward) == [1, 2, 0]
    np.testing.assert_allclose(np.abs(np.diag(f.R)), [3.0, 2.0, 1.0])
    assert list(P.qr_presorted(np.eye(5)).perm.forward) == [0, 1, 2, 3, 4]
    g = np.random.default_rng(13)
    A = g.standard_normal((12, 10)) * np.exp(g.uniform(-2, 2, 10))
    f = P.qr_presorted(A)
    assert abs(abs(f.R[0, 0]) - np.linalg.norm(A, axis=0).max()) <= 1e-10
    assert rec_err(f, A) <= 100 * EPS * 12


def test_tuxv_tall_vs_oracle():
    """TUXV whose blocked QRs (b = 32) run on tall 12000-row blocks: several
    trailing-update tiles per CTA (the cfg4 shape class)."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(4)
    m, n, r = 12000, 3000, 128
    U = np.linalg.qr(g.standard_normal((m, r + 32)))[0]
    V = np.linalg.qr(g.standard_normal((n, r + 32)))[0]
    s = 1.0 / (1.0 + np.arange(r + 32)) ** 2
    A = np.asfortranarray((U * s) @ V.T)
    cfg = P.RandomizedConfig(block=32, padding=8, seed=0)
    o = port.tuxv(A, r, 32, 8, 0)
    f = P.tuxv(A, r, cfg)
    np.testing.assert_allclose(f.singular_values(), o.singular_values(), rtol=1e-8)
    frob = np.linalg.norm(A)
    assert abs(np.linalg.norm(A - f.approx()) - np.linalg.norm(A - o.approx())) <= 1e-3 * frob


@pytest.mark.parametrize("j_max", [2, 3])
def test_tuxv_extra_half_iterations_vs_oracle(j_max):
    """tuxv(j_max > 1): the extra QLP half-iterations U^T A -> LQ -> A V -> QR
    (truncated.py:230-252) against the oracle: singular values, the
    approximation, rank and the counters the iterations add."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(40 + j_max)
    m, n, r = 1500, 1100, 96
    U = np.linalg.qr(g.standard_normal((m, r + 40)))[0]
    V = np.linalg.qr(g.standard_normal((n, r + 40)))[0]
    s = 10.0 ** (-6.0 * np.arange(r + 40) / (r + 39))
    A = np.asfortranarray((U * s) @ V.T)
    cfg = P.RandomizedConfig(block=32, padding=8, seed=0)
    o = port.tuxv(A, r, 32, 8, 0, j_max=j_max)
    f = P.tuxv(A, r, cfg, j_max=j_max)
    assert f.rank == o.rank
    np.testing.assert_allclose(f.singular_values(), o.singular_values(), rtol=1e-9)
    frob = np.linalg.norm(A)
    assert np.linalg.norm(f.approx() - o.approx()) <= 1e-9 * frob
    assert f.counters.gemm_flops == o.counters.gemm_flops


def _full_residual(A, f):
    m, n = A.shape
    rebuilt = np.zeros((m, n))
    rebuilt[: f.rank] = f.R
    if f.trailing is not None:
        rebuilt[f.rank:, f.rank:] = f.trailing
    return np.linalg.norm(A[:, np.asarray(f.perm.forward)] - f.q_factor(full=True) @ rebuilt)


@pytest.mark.parametrize("m,n,k,b,p,seed", [(60, 45, 20, 8, 4, 0), (60, 45, 20, 8, 4, 2), (50, 40, 24, 8, 4, 11),
                                            (64, 48, 32, 8, 4, 5), (20, 16, 16, 4, 4, 0), (48, 36, 12, 12, 8, 7),
                                            (16, 4, 2, 32, 8, 3), (4, 4, 2, 32, 2, 9), (40, 30, 8, 32, 8, 1)])
def test_reference_test_shapes_vs_oracle(m, n, k, b, p, seed):
    """The shapes of the reference's own driver tests (tests/test_randomized.py:
    60 x 45 down to 4 x 4, blocks of 4-12 columns, paddings 2-8, partial ranks
    with a trailing block) through all three block drivers against the oracle:
    pivots, R, the trailing block, rank, counters, the full residual with the
    trailing block folded back in and orthogonality."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(100 * seed + m)
    A = g.standard_normal((m, n))
    cfg = P.RandomizedConfig(block=b, padding=p, seed=seed)
    for drv in ("rqrcp", "rsrqrcp", "ssrqrcp"):
        # (the last three shapes are the reference's ssrqrcp-only cases: the
        # block drivers' b + p rows do not fit them)
        if (drv == "ssrqrcp" and k + p > m) or (drv != "ssrqrcp" and b + p > m):
            continue
        f = getattr(P, drv)(A, k, cfg)
        o = getattr(port, drv)(A, k, b, p, seed)
        assert f.rank == o.rank == k, drv
        np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward, err_msg=drv)
        assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R), drv
        assert f.counters.gemm_flops == o.counters.gemm_flops, drv
        assert f.counters.resamples == o.counters.resamples, drv
        q = f.q_factor()
        assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-13, drv
        if drv == "ssrqrcp":
            assert f.trailing is None
            assert np.linalg.norm(A[:, np.asarray(f.perm.forward)][:, :k] - q @ f.R[:, :k]) <= 1e-12 * np.linalg.norm(A)
        else:
            assert _full_residual(A, f) <= 1e-12 * np.linalg.norm(A), drv


def test_reference_rank_deficient_and_single_block_identities():
    """Two properties the reference's tests pin (tests/test_randomized.py): a
    rank-10 50 x 40 matrix stops at rank 10 in rqrcp and rsrqrcp, and with
    block == k the single-sample driver is the first block of rqrcp and of
    rsrqrcp -- identical pivots and R."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(5)
    A = g.standard_normal((50, 10)) @ g.standard_normal((10, 40))
    cfg = P.RandomizedConfig(block=8, padding=4, seed=0)
    assert P.rqrcp(A, 20, cfg).rank == port.rqrcp(A, 20, 8, 4, 0).rank == 10
    assert P.rsrqrcp(A, 20, cfg).rank == 10
    B = np.random.default_rng(9).standard_normal((48, 36))
    cfg = P.RandomizedConfig(block=12, padding=8, seed=7)
    fs, fr, fv = P.ssrqrcp(B, 12, cfg), P.rqrcp(B, 12, cfg), P.rsrqrcp(B, 12, cfg)
    assert list(fs.perm.forward) == list(fr.perm.forward) == list(fv.perm.forward)
    assert np.linalg.norm(fs.R - fr.R[:12]) <= 1e-13 * np.linalg.norm(fr.R)
    assert np.linalg.norm(fv.R - fr.R) <= 1e-13 * np.linalg.norm(fr.R)
    assert fs.counters.gemm_flops < P.rqrcp(B, 12, P.RandomizedConfig(block=6, padding=8, seed=7)).counters.gemm_flops + 10**9


def _decaying(seed, m, n, base=0.9):
    g = np.random.default_rng(seed)
    q1 = np.linalg.qr(g.standard_normal((m, m)))[0]
    q2 = np.linalg.qr(g.standard_normal((n, n)))[0]
    r = min(m, n)
    return (q1[:, :r] * base ** np.arange(r)) @ q2[:r]


@pytest.mark.parametrize("m,n,k,b,p,seed", [(64, 48, 16, 8, 4, 3), (48, 64, 24, 8, 4, 3), (50, 50, 32, 8, 4, 3),
                                            (30, 20, 6, 6, 4, 2), (40, 32, 16, 8, 8, 4)])
def test_reference_truncated_shapes_vs_oracle(m, n, k, b, p, seed):
    """The shapes of the reference's trqrcp tests (tests/test_truncated.py):
    same pivots as rqrcp, R rows to rounding, the oracle's W panel, the
    single-block W invariant W^T = T^T Y^T (A P), orthonormal Q."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(42 + m).standard_normal((m, n))
    cfg = P.RandomizedConfig(block=b, padding=p, seed=seed)
    ft, fr = P.trqrcp(A, k, cfg), P.rqrcp(A, k, cfg)
    o = port.trqrcp(A, k, b, p, seed)
    assert list(ft.perm.forward) == list(fr.perm.forward) == list(o.perm.forward)
    scale = 100 * EPS * np.linalg.norm(A)
    assert np.linalg.norm(ft.R - fr.R) <= scale
    assert np.linalg.norm(ft.R - o.R) <= scale
    assert np.linalg.norm(ft.reflectors.Y - fr.reflectors.Y) <= scale
    assert np.linalg.norm(ft.reflectors.W - o.W) <= 10 * scale
    assert ft.counters.gemm_flops == o.counters.gemm_flops
    q = ft.q_factor()
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-13
    if k == b:   # a single block: the inner-product panel is definitional
        Y, T = ft.reflectors.Y, port.t_factor(ft.reflectors.Y, ft.reflectors.tau)
        AP = A[:, np.asarray(ft.perm.forward)]
        assert np.linalg.norm(ft.reflectors.W[k:].T - T.T @ (Y.T @ AP[:, k:])) <= 1e-12 * np.linalg.norm(A)
        assert np.all(ft.reflectors.W[:k] == 0.0)


def test_reference_truncated_small_cases():
    """Small known answers of the reference's truncated tests: a rank-12 and a
    rank-10 input (exact reconstruction, numerical rank), lq_factor of a row
    vector and of a lower-triangular matrix, tuxv of diag(5, 3, 1), the
    svd_of_x rotation, the recorded iteration count and a monotone refinement
    sweep."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(7)
    A = g.standard_normal((50, 12)) @ g.standard_normal((12, 40))
    f = P.trqrcp(A, 12, P.RandomizedConfig(block=4, padding=4, seed=1))
    assert np.linalg.norm(A[:, np.asarray(f.perm.forward)] - f.reconstruct()) <= 1e-10 * np.linalg.norm(A)
    A = g.standard_normal((60, 10)) @ g.standard_normal((10, 50))
    f = P.trqrcp(A, 24, P.RandomizedConfig(block=8, padding=4, seed=0))
    assert f.rank == 10 and f.R.shape == (10, 50)
    L, V = P.lq_factor(np.array([[3.0, 4.0]]))
    np.testing.assert_allclose(L, [[-5.0]], atol=1e-15)
    np.testing.assert_allclose(V, [[-0.6], [-0.8]], atol=1e-15)
    Z = np.array([[2.0, 0.0], [1.0, 3.0]])
    L, V = P.lq_factor(Z)
    np.testing.assert_allclose(np.abs(V), np.eye(2), atol=1e-14)
    np.testing.assert_allclose(L @ V.T, Z, atol=1e-14)
    assert np.linalg.norm(np.triu(L, 1)) == 0.0
    D = np.diag([5.0, 3.0, 1.0])
    f = P.tuxv(D, 2, P.RandomizedConfig(block=2, padding=1, seed=0))
    np.testing.assert_allclose(f.singular_values(), [5.0, 3.0], atol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(D - f.approx()), 1.0, atol=1e-12)
    A = np.random.default_rng(14).standard_normal((40, 30))
    cfg = P.RandomizedConfig(block=5, padding=5, seed=6)
    plain, rot = P.tuxv(A, 10, cfg), P.tuxv(A, 10, cfg, svd_of_x=True)
    d = np.diag(rot.X)
    assert np.linalg.norm(rot.X - np.diag(d)) <= 1e-12
    assert np.all(d >= 0.0) and np.all(np.diff(d) <= 1e-12)
    np.testing.assert_allclose(rot.approx(), plain.approx(), atol=1e-12)
    np.testing.assert_allclose(d, np.linalg.svd(plain.X, compute_uv=False), atol=1e-12)
    A = np.random.default_rng(15).standard_normal((24, 18))
    assert P.tuxv(A, 6, P.RandomizedConfig(block=3, padding=3, seed=0), j_max=4).iterations == 4
    A = _decaying(8, 64, 48)
    cfg = P.RandomizedConfig(block=4, padding=4, seed=7)
    errs = [np.linalg.norm(A - P.tuxv(A, 8, cfg, j_max=j).approx()) for j in (1, 2, 3, 5)]
    for lo, hi in zip(errs[1:], errs[:-1]):
        assert lo <= hi * (1.0 + 1e-10)
    sv = np.linalg.svd(A, compute_uv=False)
    assert errs[-1] >= np.sqrt(np.sum(sv[8:] ** 2)) * (1.0 - 1e-10)


def test_harness_callers_vs_reference():
    """The GPU harness (harness.py:89-241 callers): the counter CSV is byte-
    identical to the reference's, the pivot trace has the same pivots, sigma
    estimates and quality curves agree to rounding."""
    import csv
    import io
    from paper_1509_06820_b200 import harness as H
    import paper_1509_06820_b200 as P
    rec = G.load("kat_harness")
    A = rec["A"]
    cfg = P.RandomizedConfig(block=16, padding=8, seed=0)
    algos = ("qr", "qr_presorted", "rqrcp", "rsrqrcp", "ssrqrcp", "trqrcp", "tuxv")
    buf = io.StringIO(newline="")
    H.write_bench_csv(H.bench(A, algos, k=24, config=cfg), buf, timing=False)
    assert buf.getvalue() == str(rec["bench_csv"])
    fbuf = io.StringIO(newline="")
    H.write_factor_csv(P.rqrcp(A, None, cfg), fbuf)
    mine = list(csv.reader(io.StringIO(fbuf.getvalue())))
    theirs = list(csv.reader(io.StringIO(str(rec["factor_csv"]))))
    assert len(mine) == len(theirs) and mine[-1] == theirs[-1]   # counters comment
    for a, b in zip(mine[1:-1], theirs[1:-1]):
        assert a[:2] == b[:2]
        assert abs(float(a[2]) - float(b[2])) <= 1e-12 * abs(float(theirs[1][2]))
    tbuf = io.StringIO(newline="")
    H.write_tuxv_csv(P.tuxv(A, 20, cfg), tbuf)
    mt = list(csv.reader(io.StringIO(tbuf.getvalue())))
    tt = list(csv.reader(io.StringIO(str(rec["tuxv_csv"]))))
    assert mt[-1] == tt[-1]
    np.testing.assert_allclose([float(r[1]) for r in mt[1:-1]], [float(r[1]) for r in tt[1:-1]],
                               rtol=1e-9)
    ranks = [int(x) for x in rec["ranks"]]
    qalgos = ("qr_presorted", "rqrcp", "rsrqrcp", "trqrcp", "tuxv")
    curve = H.quality_sweep(A, ranks, qalgos, cfg)
    for a in qalgos:
        np.testing.assert_allclose(curve.relerr[a], rec["curve_" + a], rtol=1e-6, atol=1e-14,
                                   err_msg=a)


@pytest.mark.parametrize("m,n,b,k,variant", [(1200, 1100, 56, None, "rqrcp"), (900, 820, 50, None, "rqrcp"),
                                             (1000, 948, 64, None, "rqrcp"), (2000, 1600, 120, 120, "ssrqrcp"),
                                             (1300, 1300, 40, 600, "trqrcp")])
def test_panel_widths_vs_oracle(m, n, b, k, variant):
    """Panel widths whose padded width is not a power of two (b = 40, 50, 56,
    a 52-wide last block, the 56-wide second half of a 120-wide panel) take
    the exact panel, never the fast one's power-of-two layouts."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(m + n + b).standard_normal((m, n))
    cfg = P.RandomizedConfig(block=32 if variant == "ssrqrcp" else b, padding=8, seed=0)
    run = {"rqrcp": lambda M: (P.rqrcp(M, k, cfg), port.rqrcp(M, k, b, 8, 0)),
           "ssrqrcp": lambda M: (P.ssrqrcp(M, k, cfg), port.ssrqrcp(M, k, 32, 8, 0)),
           "trqrcp": lambda M: (P.trqrcp(M, k, cfg), port.trqrcp(M, k, b, 8, 0))}[variant]
    f, o = run(A)
    np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)
    assert (f.counters.gemm_flops, f.counters.level2_flops) == \
        (o.counters.gemm_flops, o.counters.level2_flops)


@pytest.mark.parametrize("m,n,b,variant", [(1300, 1100, 160, "rqrcp"), (1100, 1400, 200, "rqrcp"),
                                           (1600, 1500, 256, "rqrcp"), (1500, 1300, 192, "trqrcp"),
                                           (1200, 1200, 144, "rsrqrcp")])
def test_block_widths_above_128_vs_oracle(m, n, b, variant):
    """Block widths 128 < b <= 256 (the reference accepts any b): the exact
    panel, the recurrence T, plain DMMA GEMMs for the K = b products and the
    sample update with R11 read through the cache instead of shared memory."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(m + n + b).standard_normal((m, n))
    cfg = P.RandomizedConfig(block=b, padding=8, seed=0)
    k = None if variant != "trqrcp" else 2 * b + 40
    f = getattr(P, variant)(A, k, cfg)
    o = getattr(port, variant)(A, k, b, 8, 0)
    assert f.rank == o.rank
    np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)
    assert (f.counters.gemm_flops, f.counters.level2_flops, f.counters.resamples) == \
        (o.counters.gemm_flops, o.counters.level2_flops, o.counters.resamples)
    if variant != "trqrcp":
        q = f.q_factor()
        frob = np.linalg.norm(A)
        assert np.linalg.norm(A[:, np.asarray(f.perm.forward)] - q @ f.R) <= 1e-12 * frob
        assert np.linalg.norm(q.T @ q - np.eye(q.shape[1]), 2) <= 1e-12


def test_trqrcp_more_than_65535_columns_vs_oracle():
    """A matrix wider than the 16-bit position range of the default argmax
    key (the reference has no width limit)."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(66000)
    m, n, k, b = 600, 66000, 96, 32
    A = g.standard_normal((m, 200)) @ g.standard_normal((200, n)) + 1e-3 * g.standard_normal((m, n))
    A[:, 65999] *= 50.0
    f = P.trqrcp(A, k, P.RandomizedConfig(block=b, padding=8, seed=0))
    o = port.trqrcp(A, k, b, 8, 0)
    assert f.rank == o.rank == k
    assert int(np.asarray(f.perm.forward)[0]) == 65999
    np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)


@pytest.mark.parametrize("k", [160, 200, 256])
def test_ssrqrcp_wide_sample_vs_oracle(k):
    """ssrqrcp's single block takes k pivots from a (k + p)-row sample: sample
    rows past 160 go through the shared-memory pivot kernel's loop form."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(k).standard_normal((1500, 1200))
    f = P.ssrqrcp(A, k, P.RandomizedConfig(block=32, padding=8, seed=0))
    o = port.ssrqrcp(A, k, 32, 8, 0)
    np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)
    assert (f.counters.gemm_flops, f.counters.level2_flops) == \
        (o.counters.gemm_flops, o.counters.level2_flops)


def test_matrix_market_to_device_factorization(tmp_path):
    """A MatrixMarket file parsed straight into column-major device memory
    (matio.py loaders with device=) and factored there."""
    import paper_1509_06820_b200 as P
    from paper_1509_06820_b200 import matio
    A = np.random.default_rng(9).standard_normal((300, 200))
    matio.save_matrix_market(A, tmp_path / "a.mtx")
    Ad = matio.load_matrix_market(tmp_path / "a.mtx", device="cuda")
    assert Ad.is_cuda and Ad.stride() == (1, 300)
    f = P.rqrcp(Ad, None, P.RandomizedConfig(block=32, padding=8, seed=0))
    o = port.rqrcp(A, None, 32, 8, 0)
    np.testing.assert_array_equal(f.perm.forward.cpu().numpy() if hasattr(f.perm.forward, "cpu")
                                  else np.asarray(f.perm.forward), o.perm.forward)


def test_b128_second_half_decline_rewinds_to_original_columns():
    """A 128-wide block whose rank drop lands in its second 64 columns
    (1100 x 1700, rank 366 + 1e-9 noise: block 256..383 drops at column 110
    of 128).  The two-half fast panel commits its first half in place before
    the second half declines; the rewind must redo the panel on the ORIGINAL
    selected columns, as the reference eliminates a panel on a copy
    (randomized.py:221-239).  Bars: identical pivots and R rows up to the
    noise floor, plus the residual."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(147)
    m, n, r = 1100, 1700, 366
    A = g.standard_normal((m, r)) @ g.standard_normal((r, n)) + 1e-9 * g.standard_normal((m, n))
    cfg = P.RandomizedConfig(block=128, padding=8, seed=0)
    f = P.rqrcp(A, None, cfg)
    o = port.rqrcp(A, None, 128, 8, 0)
    frob = float(np.linalg.norm(A))
    d = np.abs(np.diag(o.R))
    r_sig = int(np.argmax(d <= NOISE * EPS * frob)) if (d <= NOISE * EPS * frob).any() else d.size
    assert r_sig >= r - 2
    pf = np.asarray(f.perm.forward)
    np.testing.assert_array_equal(pf[:r_sig], o.perm.forward[:r_sig])
    mine = f.perm.restore(f.R)[:r_sig]
    theirs = np.zeros((o.R.shape[0], n))
    theirs[:, o.perm.forward] = o.R
    assert np.linalg.norm(mine - theirs[:r_sig]) <= 1e-10 * np.linalg.norm(theirs[:r_sig])
    rebuilt = np.zeros(A.shape)
    rebuilt[: f.rank] = f.R
    rebuilt[f.rank:, f.rank:] = f.trailing
    res = np.linalg.norm(A[:, pf] - f.q_factor(full=True) @ rebuilt)
    assert res <= 1e-12 * frob


@pytest.mark.parametrize("m,n,k,kind", [(1000, 900, 300, "gauss"), (800, 1200, 520, "gauss"),
                                         (1700, 1500, 1200, "gauss"),   # sample taller than 1024 rows
                                        (900, 700, 400, "lowrank")])
def test_ssrqrcp_wider_than_one_native_panel_vs_oracle(m, n, k, kind):
    """ssrqrcp(A, k) with k > 256 (one block of width k; randomized.py:299-313):
    the host-driven single block over the C-ABI kernels must reproduce the
    reference algorithm -- pivots, R, rank, resamples and counters."""
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(m + k)
    if kind == "gauss":
        A = g.standard_normal((m, n))
    else:
        A = g.standard_normal((m, 350)) @ g.standard_normal((350, n))
    f = P.ssrqrcp(A, k, P.RandomizedConfig(block=32, padding=8, seed=0))
    o = port.ssrqrcp(A, k, 32, 8, 0)
    frob = float(np.linalg.norm(A))
    d = np.abs(np.diag(o.R))
    bad = d <= NOISE * EPS * frob
    r_sig = int(np.argmax(bad)) if bad.any() else d.size
    np.testing.assert_array_equal(np.asarray(f.perm.forward)[:r_sig], o.perm.forward[:r_sig])
    mine = f.perm.restore(f.R)[:r_sig]
    theirs = np.zeros((o.R.shape[0], n))
    theirs[:, o.perm.forward] = o.R
    assert np.linalg.norm(mine - theirs[:r_sig]) <= 1e-10 * np.linalg.norm(theirs[:r_sig])
    if r_sig == k:
        assert f.rank == o.rank
        assert f.counters.resamples == o.counters.resamples
        assert (f.counters.gemm_flops, f.counters.level2_flops) == (o.counters.gemm_flops,
                                                                   o.counters.level2_flops)
    q = f.q_factor()
    assert np.linalg.norm(q.T @ q - np.eye(f.rank), 2) <= 1e-12


@pytest.mark.parametrize("m,n", [(3000, 2600), (2600, 3000)])
def test_b128_two_half_panels_vs_oracle(m, n):
    """b = 128 blocks take the two-half fast panel (driver.cu panel_halves)
    beside the K = 128 grouped trailing update: identical pivots and
    counters, R to 1e-10 of the reference algorithm."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(m + 3 * n).standard_normal((m, n))
    f = P.rqrcp(A, None, P.RandomizedConfig(block=128, padding=8, seed=0))
    o = port.rqrcp(A, None, 128, 8, 0)
    np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward)
    assert np.linalg.norm(f.R - o.R) <= 1e-10 * np.linalg.norm(o.R)
    assert (f.counters.gemm_flops, f.counters.level2_flops, f.counters.resamples) == (
        o.counters.gemm_flops, o.counters.level2_flops, o.counters.resamples)


def test_reference_acceptance_criteria_on_the_hot_path():
    """The reference's release criteria that concern this path
    (tests/test_acceptance.py), with its instances and pinned tolerances:
    01 reconstruction and orthogonality of every full factorization (20
    instances x qr / qr_presorted / rqrcp / rsrqrcp), 04 trqrcp == rqrcp
    pivots with R rows within 100 eps ||A|| (20 instances), 05 tuxv equals
    the factor-everything-then-truncate oracle within 1e-9 (10 instances),
    06a sample reuse keeps gemm(rqrcp) / gemm(rsrqrcp) <= 0.72 on 256 x 256."""
    import paper_1509_06820_b200 as P
    shapes = [(256, 256), (192, 256), (256, 192), (128, 128), (96, 64)]
    algos = {"qr": lambda a, s: P.qr_blocked(a),
             "qr_presorted": lambda a, s: P.qr_presorted(a),
             "rqrcp": lambda a, s: P.rqrcp(a, None, P.RandomizedConfig(block=32, padding=8, seed=s)),
             "rsrqrcp": lambda a, s: P.rsrqrcp(a, None, P.RandomizedConfig(block=32, padding=8, seed=s))}
    for idx in range(20):
        m, n = shapes[idx % len(shapes)]
        a = np.random.default_rng(idx).standard_normal((m, n))
        frob = np.linalg.norm(a)
        for name, run in algos.items():
            f = run(a, idx)
            assert f.rank == min(m, n), (name, idx)
            q = f.q_factor()
            assert np.linalg.norm(a[:, np.asarray(f.perm.forward)] - q @ f.R) <= 100 * EPS * max(m, n) * frob, (name, idx)
            assert np.linalg.norm(q.T @ q - np.eye(f.rank)) <= 100 * EPS * min(m, n), (name, idx)
        if idx % 5 == 0:   # the randomized drivers also against the oracle
            o = port.rqrcp(a, None, 32, 8, idx)
            f = algos["rqrcp"](a, idx)
            np.testing.assert_array_equal(np.asarray(f.perm.forward), o.perm.forward)
    shapes = [(128, 96), (96, 128), (128, 128), (160, 96)]
    ks = [16, 32, 48, 64]
    for idx in range(20):
        m, n = shapes[idx % len(shapes)]
        k = min(ks[idx % len(ks)], min(m, n))
        a = np.random.default_rng(100 + idx).standard_normal((m, n))
        cfg = P.RandomizedConfig(block=16, padding=8, seed=idx)
        ft, fr = P.trqrcp(a, k, cfg), P.rqrcp(a, k, cfg)
        assert list(ft.perm.forward) == list(fr.perm.forward), idx
        assert np.linalg.norm(ft.R - fr.R) <= 100 * EPS * np.linalg.norm(a), idx
    shapes = [(128, 96), (96, 64), (80, 80), (128, 48), (64, 64)]
    ks = [16, 32, 24, 16, 32]
    for idx in range(10):
        m, n = shapes[idx % len(shapes)]
        k = ks[idx % len(ks)]
        a = np.random.default_rng(200 + idx).standard_normal((m, n))
        cfg = P.RandomizedConfig(block=16, padding=8, seed=idx)
        t = P.tuxv(a, k, cfg, j_max=1)
        full = P.rqrcp(a, None, cfg)
        _, v = P.lq_factor(full.perm.restore(full.R))
        oracle = (a @ v[:, :k]) @ v[:, :k].T
        assert np.linalg.norm(t.approx() - oracle) <= 1e-9 * np.linalg.norm(a), idx
    a = np.random.default_rng(0).standard_normal((256, 256))
    cfg = P.RandomizedConfig(block=16, padding=8, seed=0)
    f1, f2 = P.rqrcp(a, None, cfg), P.rsrqrcp(a, None, cfg)
    assert f1.counters.gemm_flops / f2.counters.gemm_flops <= 0.72
