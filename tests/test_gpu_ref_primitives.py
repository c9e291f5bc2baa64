"""The reference's block-level primitives, with its signatures, on the B200:
form_reflector / apply_reflector / compose_blocks / apply_block_reflection /
downdate_norms / NormTracker (kernels.py:17-233) and SampleState /
make_sample / select_pivots / sample_update (randomized.py:48-135), against
the reference-generated known answers (tests/golden/kat_*.npz) and the oracle
(oracle/port.py, bit-identical to the reference) on the same inputs.  A last
test drives the reference's block loop (randomized.py:207-258) through these
primitives and compares with the native driver."""

import numpy as np
import pytest

from oracle import port
from tests import _golden as G

pytestmark = pytest.mark.gpu


def test_form_reflector_known_answers():
    import paper_1509_06820_b200 as P
    rec = G.load("kat_reflector")
    for i in range(6):
        x = rec[f"x{i}"]
        r = rec[f"r{i}"]
        ref = P.form_reflector(x)
        assert abs(ref.tau - r[0]) <= 1e-15 * max(1.0, abs(r[0])), i
        assert abs(ref.beta - r[1]) <= 1e-15 * max(1.0, abs(r[1])), i
        np.testing.assert_allclose(ref.v, r[2:], rtol=1e-15, atol=1e-16, err_msg=str(i))
    with pytest.raises(ValueError, match="nonempty"):
        P.form_reflector(np.zeros(0))


def test_apply_reflector_and_counters():
    import torch
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(1)
    A = g.standard_normal((70, 33))
    r = P.form_reflector(A[:, 0])
    X = A[:, 1:].copy()
    ref = X - np.outer(r.tau * r.v, r.v @ X)
    c = P.OpCounters()
    out = P.apply_reflector(X, r.v, r.tau, c)
    assert out is X
    assert np.linalg.norm(X - ref) <= 1e-14 * np.linalg.norm(ref)
    assert (c.level2_flops, c.bytes_touched) == (4 * 70 * 32, 2 * 8 * 70 * 32)
    # device operands are updated in place on the device
    Xd = torch.from_numpy(np.asfortranarray(A[:, 1:])).cuda()
    P.apply_reflector(Xd, torch.from_numpy(r.v).cuda(), r.tau)
    assert np.linalg.norm(Xd.cpu().numpy() - ref) <= 1e-14 * np.linalg.norm(ref)
    # tau = 0 and empty blocks are no-ops, as in the reference
    Z = A[:, :0]
    assert P.apply_reflector(Z, r.v, r.tau) is Z


def test_block_reflection_and_compose_vs_reference_formulas():
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(2)
    m = 90
    # reflectors of two consecutive panels, as the reference builds them
    M = g.standard_normal((m, 20))
    Y = np.zeros((m, 20))
    tau = np.zeros(20)
    for j in range(20):
        r = P.form_reflector(M[j:, j])
        Y[j:, j] = r.v
        tau[j] = r.tau
        M[j:, j + 1:] -= np.outer(r.tau * r.v, r.v @ M[j:, j + 1:])
    T1 = port.t_factor(Y[:, :12], tau[:12])
    T2 = port.t_factor(Y[:, 12:], tau[12:])
    Yc, Tc = P.compose_blocks(Y[:, :12], T1, Y[:, 12:], T2)
    T_ref = np.zeros((20, 20))
    T_ref[:12, :12], T_ref[12:, 12:] = T1, T2
    T_ref[:12, 12:] = -T1 @ ((Y[:, :12].T @ Y[:, 12:]) @ T2)
    np.testing.assert_array_equal(Yc, Y)
    assert np.linalg.norm(Tc - T_ref) <= 1e-13 * np.linalg.norm(T_ref)
    # composed T equals the single-block T of the whole reflector set
    assert np.linalg.norm(Tc - port.t_factor(Y, tau)) <= 1e-12 * np.linalg.norm(Tc)
    A = g.standard_normal((m, 45))
    for transpose in (False, True):
        X = A.copy()
        c = P.OpCounters()
        P.apply_block_reflection(X, Yc, Tc, transpose=transpose, counters=c)
        W = (Tc.T if transpose else Tc) @ (Yc.T @ A)
        ref = A - Yc @ W
        assert np.linalg.norm(X - ref) <= 1e-13 * np.linalg.norm(ref)
        assert c.gemm_flops == 4 * m * 20 * 45 + 20 * 20 * 45
    with pytest.raises(ValueError, match="row mismatch"):
        P.apply_block_reflection(np.zeros((5, 3)), Yc, Tc)


def test_downdate_norms_and_tracker_bit_identical():
    import paper_1509_06820_b200 as P
    g = np.random.default_rng(3)
    n = np.abs(g.standard_normal(300)) + 0.5
    row = g.standard_normal(300) * 0.7
    ref = np.sqrt(np.maximum(n * n - row * row, 0.0))
    np.testing.assert_array_equal(P.downdate_norms(n, row), ref)
    # the tracker reproduces the reference's (oracle's) downdates and
    # recomputes exactly the columns the sqrt(eps) guard flags
    A = np.asfortranarray(g.standard_normal((40, 64)))
    A[:, 5] = A[:, 0] * (1 + 1e-9)          # forces a cancellation -> recompute
    tr = P.NormTracker(A)
    ref_tr = port.Norms(A)
    np.testing.assert_array_equal(tr.norms, ref_tr.val)
    W = A.copy()
    for j in range(6):
        p, nrm = tr.max_trailing(j)
        q, nq = ref_tr.argmax_from(j)
        assert (p, nrm) == (q, nq)
        W[:, [j, p]] = W[:, [p, j]]
        tr.swap(j, p)
        ref_tr.swap(j, p)
        r = P.form_reflector(W[j:, j])
        W[j:, j + 1:] -= np.outer(r.tau * r.v, r.v @ W[j:, j + 1:])
        W[j, j], W[j + 1:, j] = r.beta, 0.0
        tr.downdate(j + 1, W[j, j + 1:], lambda c: W[j + 1:, c])
        ref_tr.downdate(j + 1, W[j, j + 1:], lambda c: W[j + 1:, c])
        np.testing.assert_allclose(tr.norms, ref_tr.val, rtol=1e-14, atol=0)


def test_sample_primitives_match_oracle_and_known_answers():
    import paper_1509_06820_b200 as P
    # select_pivots on the reference's select known answers
    rec = G.load("kat_select")
    for key in sorted({k.rsplit("_", 1)[0] for k in rec}):
        B = rec[f"{key}_B"]
        want = int(rec[f"{key}_want"])
        smp = P.SampleState(B=np.asfortranarray(B.copy()), ell=B.shape[0])
        c = P.OpCounters()
        perm, got = P.select_pivots(smp, want, c)
        assert got == int(rec[f"{key}_got"]), key
        np.testing.assert_array_equal(perm.forward, rec[f"{key}_perm"], err_msg=key)
        np.testing.assert_array_equal(np.array(perm.swaps).reshape(-1, 2), rec[f"{key}_swaps"])
        scale = float(np.linalg.norm(B))
        assert np.linalg.norm(smp.B - rec[f"{key}_S"]) <= 1e-12 * scale, key
        assert c.level2_flops == int(rec[f"{key}_l2"]), key
        assert smp.s11.shape == (got, got) and smp.s22.shape == (B.shape[0] - got, B.shape[1] - got)
    with pytest.raises(ValueError, match="cannot select 9 pivots"):
        P.select_pivots(P.SampleState(B=np.ones((4, 6)), ell=4), 9)

    # make_sample / select_pivots / sample_update vs the oracle, same stream
    g = np.random.default_rng(4)
    A = g.standard_normal((300, 220))
    ell, b = 24, 16
    s_gpu = P.make_sample(A, ell, P.RngState(7), c_gpu := P.OpCounters())
    s_ref = port.sketch(A, ell, port.Stream(7), c_ref := port.Counters())
    assert np.linalg.norm(s_gpu.B - s_ref.B) <= 1e-13 * np.linalg.norm(s_ref.B)
    assert abs(s_gpu.frob_a - s_ref.frob_a) <= 1e-14 * s_ref.frob_a
    assert (c_gpu.gemm_flops, c_gpu.bytes_touched) == (c_ref.gemm_flops, c_ref.bytes_touched)
    s_gpu.B = s_ref.B.copy()                 # identical bytes from here on
    perm_g, got_g = P.select_pivots(s_gpu, b)
    perm_r, got_r = port.pick_pivots(s_ref, b, port.Counters())
    assert got_g == got_r == b
    np.testing.assert_array_equal(perm_g.forward, perm_r.forward)
    # the panel on the chosen columns, then the sample downdate
    W = A[:, perm_g.forward].copy()
    Rfull = np.linalg.qr(W[:, :b], mode="r")
    R12 = np.linalg.qr(W[:, :b])[0].T @ W[:, b:]
    c1, c2 = P.OpCounters(), port.Counters()
    P.sample_update(s_gpu, Rfull, R12, c1)
    port.downdate_sample(s_ref, Rfull, R12, c2)
    assert np.linalg.norm(s_gpu.B - s_ref.B) <= 1e-12 * np.linalg.norm(s_ref.B)
    assert (c1.gemm_flops, c1.bytes_touched) == (c2.gemm_flops, c2.bytes_touched)
    assert s_gpu.block == 1 and s_gpu.s11 is None
    with pytest.raises(ValueError, match="no matching factorization"):
        P.sample_update(s_gpu, Rfull, R12)
    # a singular block triangle raises DegenerateSampleError
    s3 = P.make_sample(A, ell, P.RngState(7))
    P.select_pivots(s3, b)
    Rbad = Rfull.copy()
    Rbad[3, 3] = 0.0
    with pytest.raises(P.DegenerateSampleError):
        P.sample_update(s3, Rbad, R12)


def test_reference_block_loop_through_the_primitives():
    """The reference's _randomized_factor loop (randomized.py:207-258) written
    against the drop-in primitives reproduces the native driver's pivots."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(9).standard_normal((160, 130))
    cfg = P.RandomizedConfig(block=16, padding=8, seed=0)
    work = np.array(A, order="F")
    m, n = work.shape
    rng = P.RngState(cfg.seed)
    frob = float(np.linalg.norm(work))
    perm = P.Permutation.identity(n)
    smp = P.make_sample(work, cfg.ell, rng)
    smp.frob_a = frob
    i0 = 0
    while i0 < n:
        want = min(cfg.block, n - i0)
        lp, got = P.select_pivots(smp, want)
        assert got == want
        for a_, c_ in lp.swaps:
            perm.swap(i0 + a_, i0 + c_)
            if a_ != c_:
                work[:, [i0 + a_, i0 + c_]] = work[:, [i0 + c_, i0 + a_]]
        panel = work[i0:, i0:i0 + got].copy()
        Y = np.zeros_like(panel)
        tau = np.zeros(got)
        for j in range(got):
            r = P.form_reflector(panel[j:, j])
            Y[j:, j], tau[j] = r.v, r.tau
            P.apply_reflector(panel[j:, j + 1:], r.v, r.tau)
            panel[j, j], panel[j + 1:, j] = r.beta, 0.0
        work[i0:, i0:i0 + got] = panel
        T = P.build_t_matrix(Y, tau)
        C = work[i0:, i0 + got:]
        if C.shape[1]:
            C = np.array(C, order="F")
            P.apply_block_reflection(C, Y, T, transpose=True)
            work[i0:, i0 + got:] = C
        i0 += got
        if i0 < n:
            P.sample_update(smp, work[i0 - got:i0, i0 - got:i0], work[i0 - got:i0, i0:])
    f = P.rqrcp(A, None, cfg)
    np.testing.assert_array_equal(perm.forward, f.perm.forward)
    assert np.linalg.norm(work[:min(m, n)] - f.R) <= 1e-11 * np.linalg.norm(f.R)


def test_reference_sample_primitive_small_cases():
    """Small properties the reference's own tests pin for the sample
    primitives (tests/test_randomized.py), at their sizes: one GEMM's counters
    and shapes, a zero matrix, ell validation, descending-norm selection on a
    diagonal sample, the definitional QRCP of a square sample, R12 = 0 keeps
    S12 and S22 bit for bit, a 1e-300 diagonal raises."""
    import paper_1509_06820_b200 as P
    A = np.random.default_rng(0).standard_normal((12, 9))
    c = P.OpCounters()
    s = P.make_sample(A, 6, P.RngState(3), c)
    assert s.B.shape == (6, 9) and s.ell == 6
    assert c.gemm_flops == 2 * 6 * 12 * 9
    assert np.all(P.make_sample(np.zeros((5, 4)), 3, P.RngState(0), P.OpCounters()).B == 0.0)
    with pytest.raises(ValueError):
        P.make_sample(np.eye(4), 0, P.RngState(0), P.OpCounters())
    B = np.zeros((4, 6))
    np.fill_diagonal(B, [2.0, 5.0, 1.0, 4.0])
    smp = P.SampleState(B=B.copy(), ell=4, frob_a=float(np.linalg.norm(B)))
    perm, got = P.select_pivots(smp, 4, P.OpCounters())
    assert got == 4 and list(perm.forward[:4]) == [1, 3, 0, 2]
    # square sample, all pivots: the eliminated sample carries the QRCP's R
    B = np.random.default_rng(7).standard_normal((5, 5))
    smp = P.SampleState(B=B.copy(), ell=5, frob_a=float(np.linalg.norm(B)))
    perm, got = P.select_pivots(smp, 5, P.OpCounters())
    ref = port.Sample(B=np.asfortranarray(B.copy()), ell=5)
    perm_r, got_r = port.pick_pivots(ref, 5, port.Counters())
    assert got == got_r == 5 and list(perm.forward) == list(perm_r.forward)
    assert np.linalg.norm(np.triu(smp.B) - np.triu(ref.B)) <= 1e-12 * np.linalg.norm(B)
    Qr = np.linalg.qr(B[:, perm.forward], mode="r")
    assert np.linalg.norm(np.abs(np.triu(smp.B)) - np.abs(Qr)) <= 1e-12 * np.linalg.norm(B)
    # R12 = 0: the correction vanishes exactly
    g = np.random.default_rng(1)
    B = g.standard_normal((5, 8))
    smp = P.SampleState(B=B.copy(), ell=5, frob_a=float(np.linalg.norm(B)))
    _, got = P.select_pivots(smp, 2, P.OpCounters())
    assert got == 2
    s12, s22 = smp.s12.copy(), smp.s22.copy()
    r11 = np.triu(g.standard_normal((2, 2))) + 5.0 * np.eye(2)
    P.sample_update(smp, r11, np.zeros((2, 6)), P.OpCounters())
    np.testing.assert_array_equal(smp.B[:2], s12)
    np.testing.assert_array_equal(smp.B[2:], s22)
    g = np.random.default_rng(2)
    B = g.standard_normal((4, 6))
    smp = P.SampleState(B=B.copy(), ell=4, frob_a=float(np.linalg.norm(B)))
    P.select_pivots(smp, 2, P.OpCounters())
    with pytest.raises(P.DegenerateSampleError):
        P.sample_update(smp, np.array([[1.0, 0.5], [0.0, 1e-300]]), g.standard_normal((2, 4)),
                        P.OpCounters())


def test_reference_select_quality_monte_carlo():
    """The reference's replay check (tests/test_randomized.py): 200 seeded
    6 x 10 samples, 4 pivots each; every pick must be the argmax of the
    independently recomputed residual norms (within the 0.5x floor the
    reference uses), and equal the oracle's pick."""
    import paper_1509_06820_b200 as P
    good = 0
    for t in range(200):
        B = np.random.default_rng(t).standard_normal((6, 10))
        smp = P.SampleState(B=B.copy(), ell=6, frob_a=float(np.linalg.norm(B)))
        perm, got = P.select_pivots(smp, 4, P.OpCounters())
        assert got == 4
        ref = port.Sample(B=np.asfortranarray(B.copy()), ell=6)
        perm_r, _ = port.pick_pivots(ref, 4, port.Counters())
        assert list(perm.forward) == list(perm_r.forward), t
        work = B[:, perm.forward].copy()
        ok = True
        for step in range(4):
            norms = np.sum(work[step:, step:] ** 2, axis=0)
            ok = ok and norms[0] >= 0.5 * norms.max()
            v, tau, beta = port.householder(work[step:, step].copy())
            work[step, step] = beta
            work[step + 1:, step] = 0.0
            port.reflect_left(work[step:, step + 1:], v, tau)
        good += ok
    assert good == 200


def test_reference_kernel_small_known_answers():
    """The reference's small known answers for the block kernels
    (tests/test_kernels.py): [3, 4] -> beta -5, tau 1.6, v [1, 0.5]; an
    aligned vector still flips; the zero vector; T of one reflector and of
    orthogonal reflectors; empty and mismatched compose_blocks; the block
    reflection's round trip, flop count and no-op cases; column norms of the
    identity; norm downdates 5, 4 -> 3 and never negative."""
    import paper_1509_06820_b200 as P
    r = P.form_reflector(np.array([3.0, 4.0]))
    assert r.beta == -5.0 and abs(r.tau - 1.6) <= 1e-15
    np.testing.assert_allclose(r.v, [1.0, 0.5])
    H = np.eye(2) - r.tau * np.outer(r.v, r.v)
    np.testing.assert_allclose(H @ [3.0, 4.0], [-5.0, 0.0], atol=1e-14)
    r2 = P.form_reflector(np.array([2.0, 0.0, 0.0]))
    assert r2.tau == 2.0 and r2.beta == -2.0
    np.testing.assert_allclose(r2.v, [1.0, 0.0, 0.0])
    r0 = P.form_reflector(np.zeros(2))
    assert r0.tau == 0.0 and r0.beta == 0.0 and r0.v[0] == 1.0
    # involution and annihilation on random vectors
    for n, seed in ((1, 0), (7, 3), (40, 9)):
        x = np.random.default_rng(seed).standard_normal(n)
        rr = P.form_reflector(x)
        H = np.eye(n) - rr.tau * np.outer(rr.v, rr.v)
        e1 = np.zeros(n); e1[0] = rr.beta
        assert np.linalg.norm(H @ x - e1) <= 1e-13 * max(1.0, np.linalg.norm(x))
        assert np.linalg.norm(H @ H - np.eye(n)) <= 1e-13
    np.testing.assert_allclose(P.build_t_matrix(r.v.reshape(2, 1), np.array([r.tau])), [[r.tau]])
    Y = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 0.0], [0.0, 2.0]])
    tau = 2.0 / np.sum(Y * Y, axis=0)
    np.testing.assert_allclose(P.build_t_matrix(Y, tau), np.diag(tau), atol=1e-15)
    g = np.random.default_rng(4)
    Y3, T3 = g.standard_normal((8, 3)), g.standard_normal((3, 3))
    Yc, Tc = P.compose_blocks(Y3, T3, np.zeros((8, 0)), np.zeros((0, 0)))
    np.testing.assert_allclose(Yc, Y3)
    np.testing.assert_allclose(Tc, T3)
    _, Tc = P.compose_blocks(np.zeros((8, 0)), np.zeros((0, 0)), Y3, T3)
    np.testing.assert_allclose(Tc, T3)
    with pytest.raises(ValueError):
        P.compose_blocks(np.ones((4, 1)), np.ones((1, 1)), np.ones((5, 1)), np.ones((1, 1)))
    # a genuine 5-reflector block on 20 rows: H then H^T is the identity
    m, n, b = 20, 9, 5
    M = np.random.default_rng(7).standard_normal((m, b))
    Yb, tb = port.panel_qr(np.asfortranarray(M.copy()))
    Tb = P.build_t_matrix(Yb, tb)
    assert np.linalg.norm(Tb - port.t_factor(Yb, tb)) <= 1e-14 * np.linalg.norm(Tb)
    A0 = np.random.default_rng(8).standard_normal((m, n))
    A = A0.copy()
    c = P.OpCounters()
    P.apply_block_reflection(A, Yb, Tb, counters=c)
    P.apply_block_reflection(A, Yb, Tb, transpose=True, counters=c)
    np.testing.assert_allclose(A, A0, atol=1e-12)
    assert c.gemm_flops == 2 * (4 * m * b * n + b * b * n) and c.bytes_touched > 0
    with pytest.raises(ValueError):
        P.apply_block_reflection(np.ones((7, 3)), Yb[:8, :2], Tb[:2, :2])
    A1 = np.ones((8, 3))
    P.apply_block_reflection(A1, np.zeros((8, 0)), np.zeros((0, 0)))
    np.testing.assert_allclose(A1, 1.0)
    np.testing.assert_allclose(P.column_norms(np.eye(4)), np.ones(4))
    assert abs(P.downdate_norms(np.array([5.0]), np.array([4.0]))[0] - 3.0) <= 1e-15
    assert P.downdate_norms(np.array([3.0]), np.array([3.0000001]))[0] == 0.0
