"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Outputs ``tests/golden/*.npz``.  Each fixture stores the inputs (or the seeded
recipe that rebuilds them) and the reference's own outputs: permutation,
swap log, R, Y, tau, W, trailing block, rank, counters and resample count.
Large outputs are stored as a sha256 of their bytes plus a few slices, so the
directory stays small.  The oracle (``oracle/port.py``) and the GPU path are
both checked against these files.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _gaussian(seed, m, n):
    return np.random.default_rng(seed).standard_normal((m, n))


def _lowrank(seed, m, n, r):
    g = np.random.default_rng(seed)
    return g.standard_normal((m, r)) @ g.standard_normal((r, n))


def _geometric(seed, n, decades):
    g = np.random.default_rng(seed)
    U = np.linalg.qr(g.standard_normal((n, n)))[0]
    V = np.linalg.qr(g.standard_normal((n, n)))[0]
    s = 10.0 ** (-decades * np.arange(n) / (n - 1))
    return np.asfortranarray((U * s) @ V.T)


def _decay(seed, m, n, base=0.9):
    g = np.random.default_rng(seed)
    q1, _ = np.linalg.qr(g.standard_normal((m, m)))
    q2, _ = np.linalg.qr(g.standard_normal((n, n)))
    r = min(m, n)
    return q1[:, :r] * (base ** np.arange(r)) @ q2[:r]


# (name, driver, A-builder, k, block, padding, seed, store_full)
CASES = [
    ("rq_gauss_60x45_k20", "rqrcp", lambda: _gaussian(0, 60, 45), 20, 8, 4, 0, True),
    ("rq_gauss_45x60_full", "rqrcp", lambda: _gaussian(1, 45, 60), None, 8, 4, 1, True),
    ("rq_gauss_64x64_full", "rqrcp", lambda: _gaussian(2, 64, 64), None, 16, 8, 2, True),
    ("rq_gauss_130x97_full", "rqrcp", lambda: _gaussian(3, 130, 97), None, 32, 8, 5, True),
    ("rq_lowrank_50x40_r10", "rqrcp", lambda: _lowrank(5, 50, 40, 10), 20, 8, 4, 0, True),
    ("rq_lowrank_80x70_r13", "rqrcp", lambda: _lowrank(6, 80, 70, 13), None, 8, 4, 3, True),
    ("rq_zero_12x9", "rqrcp", lambda: np.zeros((12, 9)), None, 4, 2, 0, True),
    ("rq_geom16_128_b8", "rqrcp", lambda: _geometric(0, 128, 16.0), None, 8, 8, 0, True),
    ("rq_geom20_192_b16", "rqrcp", lambda: _geometric(0, 192, 20.0), None, 16, 8, 0, True),
    ("rq_geom12_512_b32", "rqrcp", "geom:1:512:12", None, 32, 8, 0, False),
    ("rq_dup_cols_40x30", "rqrcp",
     lambda: np.repeat(_gaussian(7, 40, 10), 3, axis=1), None, 8, 4, 0, True),
    ("rs_gauss_64x48_k32", "rsrqrcp", lambda: _gaussian(6, 64, 48), 32, 8, 4, 5, True),
    ("rs_lowrank_50x40_r10", "rsrqrcp", lambda: _lowrank(5, 50, 40, 10), 20, 8, 4, 0, True),
    ("rs_geom16_128_b8", "rsrqrcp", lambda: _geometric(0, 128, 16.0), None, 8, 8, 0, True),
    ("ss_gauss_48x36_k12", "ssrqrcp", lambda: _gaussian(9, 48, 36), 12, 12, 8, 7, True),
    ("ss_lowrank_40x30_r8", "ssrqrcp", lambda: _lowrank(3, 40, 30, 8), 8, 32, 8, 1, True),
    ("tr_gauss_64x48_k16", "trqrcp", lambda: _gaussian(42, 64, 48), 16, 8, 4, 3, True),
    ("tr_gauss_48x64_k24", "trqrcp", lambda: _gaussian(42, 48, 64), 24, 8, 4, 3, True),
    ("tr_gauss_50x50_k32", "trqrcp", lambda: _gaussian(42, 50, 50), 32, 8, 4, 3, True),
    ("tr_lowrank_60x50_r10", "trqrcp", lambda: _lowrank(9, 60, 50, 10), 24, 8, 4, 0, True),
    ("tr_geom16_128_full", "trqrcp", lambda: _geometric(0, 128, 16.0), 128, 8, 8, 0, True),
    ("tr_geom20_192_full", "trqrcp", lambda: _geometric(0, 192, 20.0), 192, 16, 8, 0, True),
    ("tr_geom12_512_k256", "trqrcp", "geom:1:512:12", 256, 32, 8, 0, False),
    ("tx_diag_531", "tuxv", lambda: np.diag([5.0, 3.0, 1.0]), 2, 2, 1, 0, True),
    ("tx_lowrank_45x35_r9", "tuxv", lambda: _lowrank(11, 45, 35, 9), 9, 4, 4, 1, True),
    ("tx_decay_72x56_k16", "tuxv", lambda: _decay(6, 72, 56), 16, 8, 8, 3, True),
    ("tx_gauss_200x150_k40", "tuxv", lambda: _gaussian(13, 200, 150), 40, 8, 4, 2, True),
]

# config 1 of BASELINE.json: full RQRCP of a seeded 1000x1000 Gaussian
CFG1 = ("cfg1_rq_gauss_1000", "rqrcp", "gauss:0:1000:1000", None, 32, 8, 0, False)


def build_recipe(recipe):
    """Seeded recipes for the inputs that are not stored in the fixture.
    ``gauss`` is bit-portable (PCG64 + ziggurat); ``geom`` goes through
    LAPACK QR and is only bit-stable on the CPU that generated it."""
    kind, *args = recipe.split(":")
    if kind == "gauss":
        seed, m, n = map(int, args)
        return _gaussian(seed, m, n)
    if kind == "geom":
        seed, n, dec = int(args[0]), int(args[1]), float(args[2])
        return _geometric(seed, n, dec)
    raise ValueError(recipe)


def _run_reference(rq, driver, A, k, block, padding, seed):
    cfg = rq.RandomizedConfig(block=block, padding=padding, seed=seed)
    if driver == "rqrcp":
        return rq.rqrcp(A, k=k, config=cfg)
    if driver == "rsrqrcp":
        return rq.rsrqrcp(A, k=k, config=cfg)
    if driver == "ssrqrcp":
        return rq.ssrqrcp(A, k=k, config=cfg)
    if driver == "trqrcp":
        return rq.trqrcp(A, k=k, config=cfg)
    if driver == "tuxv":
        return rq.tuxv(A, k=k, config=cfg)
    raise ValueError(driver)


def _store(name, driver, A, k, block, padding, seed, full, f, recipe=""):
    rec = dict(driver=driver, k=-1 if k is None else k, block=block, padding=padding,
               seed=seed, m=A.shape[0], n=A.shape[1], full=full)
    c = f.counters
    rec.update(gemm_flops=c.gemm_flops, level2_flops=c.level2_flops,
               bytes_touched=c.bytes_touched, resamples=c.resamples, rank=f.rank)
    if driver == "tuxv":
        outs = dict(U=f.U, V=f.V, X=f.X, sv=f.singular_values())
    else:
        outs = dict(perm=np.asarray(f.perm.forward, dtype=np.int64),
                    swaps=np.asarray(f.perm.swaps, dtype=np.int64).reshape(-1, 2),
                    R=f.R, Y=f.reflectors.Y, tau=f.reflectors.tau)
        if getattr(f, "trailing", None) is not None:
            outs["trailing"] = f.trailing
        if f.reflectors.W is not None:
            outs["W"] = f.reflectors.W
    if full:
        rec["A"] = np.asarray(A)
        rec.update(outs)
    else:
        rec["recipe"] = recipe
        for key, val in outs.items():
            rec[f"sha_{key}"] = _sha(val)
        for key in ("perm", "tau", "swaps"):
            if key in outs:
                rec[key] = outs[key]
        rec["R_diag"] = np.diag(outs["R"]).copy()
        rec["R_head"] = outs["R"][:8].copy()
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **rec)


def make_qr(rq):
    # qr_blocked / qr_presorted (qrcp.py:222-268) and column_norms
    # (kernels.py:184-186); C-order and F-order inputs (numpy's norm sums in a
    # layout-dependent order), tied norms, a partial rank
    rec = {}
    g = np.random.default_rng(77)
    qcases = {
        "gaussC": (np.ascontiguousarray(g.standard_normal((120, 90))), None, 32),
        "gaussF": (np.asfortranarray(g.standard_normal((150, 70))), 50, 16),
        "lowrank": (np.ascontiguousarray(_lowrank(5, 100, 80, 12)), None, 32),
    }
    # exact ties without rank deficiency: entry sign flips keep every square
    # and its summation position, so the three copies' norms are equal bitwise
    T = g.standard_normal((64, 20))
    D1, D2 = (np.where(g.standard_normal((64, 1)) < 0, -1.0, 1.0) for _ in range(2))
    qcases["ties"] = (np.ascontiguousarray(np.hstack([T, D1 * T[:, ::-1], D2 * T])), None, 8)
    for key, (A, k, b) in qcases.items():
        ctr = rq.OpCounters()
        f = rq.qr_presorted(A, k, b, ctr)
        fb = rq.qr_blocked(A, k, b, rq.OpCounters())
        rec[f"{key}_A"] = A
        rec[f"{key}_forder"] = np.array(int(A.flags.f_contiguous and not A.flags.c_contiguous))
        rec[f"{key}_k"] = np.array(-1 if k is None else k)
        rec[f"{key}_b"] = np.array(b)
        rec[f"{key}_norms"] = rq.column_norms(A)
        rec[f"{key}_perm"] = np.asarray(f.perm.forward)
        rec[f"{key}_R"] = f.R
        rec[f"{key}_Y"] = f.reflectors.Y
        rec[f"{key}_tau"] = f.reflectors.tau
        rec[f"{key}_trailing"] = f.trailing
        rec[f"{key}_counters"] = np.array([ctr.gemm_flops, ctr.level2_flops, ctr.bytes_touched])
        rec[f"{key}_blocked_R"] = fb.R
        rec[f"{key}_blocked_counters"] = np.array([fb.counters.gemm_flops, fb.counters.level2_flops,
                                                   fb.counters.bytes_touched])
    np.savez_compressed(os.path.join(OUT, "kat_qr_presorted.npz"), **rec)


def make_harness(rq):
    """harness.py callers: counter CSV (byte-stable), pivot
    trace CSV, sigma CSV and quality curves of the reference on one
    synthetic matrix."""
    import io
    from rqrcp import harness as H
    A = H.synthetic_matrix("stepped", 120, 96, seed=3)
    cfg = rq.RandomizedConfig(block=16, padding=8, seed=0)
    algos = ("qr", "qr_presorted", "rqrcp", "rsrqrcp", "ssrqrcp", "trqrcp", "tuxv")
    buf = io.StringIO(newline="")
    H.write_bench_csv(H.bench(A, algos, k=24, config=cfg), buf, timing=False)
    fbuf = io.StringIO(newline="")
    H.write_factor_csv(rq.rqrcp(A, None, cfg), fbuf)
    tbuf = io.StringIO(newline="")
    H.write_tuxv_csv(rq.tuxv(A, 20, cfg), tbuf)
    ranks = [8, 16, 24, 32, 40]
    qalgos = ("qr_presorted", "rqrcp", "rsrqrcp", "trqrcp", "tuxv")
    curve = H.quality_sweep(A, ranks, qalgos, cfg)
    rec = {"A": A, "bench_csv": np.array(buf.getvalue()), "factor_csv": np.array(fbuf.getvalue()),
           "tuxv_csv": np.array(tbuf.getvalue()), "ranks": np.array(ranks)}
    for a in qalgos:
        rec["curve_" + a] = np.asarray(curve.relerr[a])
    np.savez_compressed(os.path.join(OUT, "kat_harness.npz"), **rec)


MATIO_CASES = {
    "mm_array": b"%%MatrixMarket matrix array real general\n2 3\n1\n2\n3\n4\n5\n6\n",
    "mm_sym": b"%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n",
    "mm_coord_dup": b"%%MatrixMarket matrix coordinate real general\n% c\n3 3 4\n1 1 1.5\n2 3 2\n"
                    b"1 1 0.25\n3 1 -1\n",
    "mm_coord_sym": b"%%MatrixMarket matrix coordinate integer symmetric\n3 3 5\n1 1 1\n2 1 2\n"
                    b"1 2 3\n3 2 4e-1\n2 1 0.1\n",
    "mm_field": b"%%MatrixMarket matrix array complex general\n2 2\n1\n2\n3\n4\n",
    "mm_count": b"%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "mm_index": b"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "mm_nan": b"%%MatrixMarket matrix array real general\n1 2\n1\nnan\n",
    "mm_header": b"%MatrixMarket matrix array real general\n1 1\n1\n",
    "mm_rect_sym": b"%%MatrixMarket matrix array real symmetric\n2 3\n1\n",
    "mm_size": b"%%MatrixMarket matrix array real general\n2 x\n",
    "mm_empty": b"",
    "mm_nosize": b"%%MatrixMarket matrix array real general\n% only comment\n",
    "mm_coord_bad": b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "pgm_p2": b"P2\n# c\n3 2\n255\n0 128 255\n1 2 3\n",
    "pgm_p5_16": b"P5\n2 2\n65535\n\x00\x01\x00\x02\xff\xff\x00\x03",
    "pgm_p5_inline": b"P5 2 1 255\n\x05\x06",
    "pgm_magic": b"P3\n1 1\n1\n1\n",
    "pgm_trunc": b"P5\n2 2\n255\n\x01\x02",
    "pgm_maxval": b"P2\n1 1\n70000\n1\n",
    "pgm_sample": b"P2\n1 1\n10\n11\n",
    "pgm_width": b"P2\nx 1\n1\n",
    "pgm_eoh": b"P2\n1",
}


def make_matio(rq):
    """matio.py loaders on valid and malformed files: the parsed matrix, or
    the error class and message (path replaced by {path})."""
    import tempfile
    from rqrcp import matio as M
    rec = {}
    d = tempfile.mkdtemp()
    for name, raw in MATIO_CASES.items():
        fn = os.path.join(d, name)
        with open(fn, "wb") as fh:
            fh.write(raw)
        rec[name + "_bytes"] = np.frombuffer(raw, dtype=np.uint8)
        try:
            out = (M.load_matrix_market if name.startswith("mm") else M.load_pgm)(fn)
            rec[name + "_out"] = out
        except ValueError as e:
            rec[name + "_err"] = np.array(type(e).__name__ + ": " + str(e).replace(fn, "{path}"))
    g = np.random.default_rng(5)
    A = g.standard_normal((7, 5))
    M.save_matrix_market(A, os.path.join(d, "save.mtx"))
    rec["save_A"] = A
    rec["save_mtx"] = np.frombuffer(open(os.path.join(d, "save.mtx"), "rb").read(), dtype=np.uint8)
    img = np.clip(g.uniform(-0.2, 1.2, (6, 9)), -1, 2)
    rec["save_img"] = img
    for asc in (0, 1):
        for mv in (255, 1000):
            fn = os.path.join(d, f"s{asc}{mv}.pgm")
            M.save_pgm(img, fn, mv, bool(asc))
            rec[f"save_pgm_{asc}_{mv}"] = np.frombuffer(open(fn, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "kat_matio.npz"), **rec)


def main():
    sys.path.insert(0, REF)
    import rqrcp as rq  # the reference package

    # Ω stream known answers (rng.py:36-41), used to pin host RNG replays
    st = rq.RngState(0)
    om40 = rq.gaussian_matrix(st, 40, 8)
    st2 = rq.RngState(0, position=40 * 8)
    tail = rq.gaussian_matrix(st2, 40, 3)
    st3 = rq.RngState(0)
    om72 = rq.gaussian_matrix(st3, 72, 2)
    np.savez_compressed(os.path.join(OUT, "kat_rng.npz"), om40=om40, tail=tail, om72=om72)

    # reflector KATs (test_kernels.py:71-98 style inputs)
    xs = [np.array([3.0, 4.0]), np.array([2.0, 0.0, 0.0]), np.zeros(3),
          np.array([-1.0, 2.0, -2.0]), np.array([0.0, 1.0]), np.array([7.0])]
    refl = []
    for x in xs:
        r = rq.form_reflector(x)
        refl.append(np.concatenate([[r.tau, r.beta], r.v]))
    np.savez_compressed(os.path.join(OUT, "kat_reflector.npz"),
                        **{f"x{i}": x for i, x in enumerate(xs)},
                        **{f"r{i}": r for i, r in enumerate(refl)})

    # select_pivots on fixed samples: diag KAT plus random samples
    samples = {}
    b = np.zeros((4, 6))
    np.fill_diagonal(b, [2.0, 5.0, 1.0, 4.0])
    samples["diag"] = (b, 4)
    for s in range(6):
        g = np.random.default_rng(100 + s)
        ell = int(g.integers(6, 20))
        nt = int(g.integers(ell, 60))
        samples[f"rand{s}"] = (g.standard_normal((ell, nt)) * g.uniform(0.1, 3.0, nt), ell - 3)
    g = np.random.default_rng(7)
    big = g.standard_normal((72, 700)) * np.exp(g.uniform(-3, 3, 700))
    samples["wide72"] = (big, 64)
    # duplicated columns force exact norm ties (first max by position)
    dup = np.repeat(np.random.default_rng(8).standard_normal((10, 5)), 4, axis=1)
    samples["ties"] = (dup, 6)
    # norm-recompute guard: columns that lie almost in the span of others
    base = np.random.default_rng(9).standard_normal((16, 6))
    near = base @ np.random.default_rng(10).standard_normal((6, 20))
    near += 1e-9 * np.random.default_rng(11).standard_normal(near.shape)
    samples["guard"] = (np.hstack([base, near]), 12)
    rec = {}
    for key, (B, want) in samples.items():
        smp = rq.SampleState(B=np.asfortranarray(B.copy()), ell=B.shape[0],
                             frob_a=float(np.linalg.norm(B)))
        ctr = rq.OpCounters()
        perm, got = rq.select_pivots(smp, want, ctr)
        rec[f"{key}_B"] = B
        rec[f"{key}_want"] = want
        rec[f"{key}_got"] = got
        rec[f"{key}_perm"] = np.asarray(perm.forward, dtype=np.int64)
        rec[f"{key}_swaps"] = np.asarray(perm.swaps, dtype=np.int64).reshape(-1, 2)
        rec[f"{key}_S"] = smp.B.copy()
        rec[f"{key}_Ys"] = smp.reflectors.Y
        rec[f"{key}_taus"] = smp.reflectors.tau
        rec[f"{key}_l2"] = ctr.level2_flops
    np.savez_compressed(os.path.join(OUT, "kat_select.npz"), **rec)

    # panel + T matrix KATs
    rec = {}
    for s, (mm, bw) in enumerate([(40, 8), (300, 32), (33, 33), (70, 5)]):
        P = np.random.default_rng(200 + s).standard_normal((mm, bw))
        if s == 3:
            P[:, 2] = 0.0  # a zero column: identity reflector
        Pc = np.asfortranarray(P.copy())
        ctr = rq.OpCounters()
        Yp, tp = rq.qrcp.panel_householder(Pc, ctr)
        rec[f"p{s}_P"] = P
        rec[f"p{s}_R"] = Pc
        rec[f"p{s}_Y"] = Yp
        rec[f"p{s}_tau"] = tp
        rec[f"p{s}_T"] = rq.build_t_matrix(Yp, tp)
        rec[f"p{s}_l2"] = ctr.level2_flops
    np.savez_compressed(os.path.join(OUT, "kat_panel.npz"), **rec)

    make_qr(rq)
    make_harness(rq)
    make_matio(rq)

    for name, driver, build, k, block, padding, seed, full in CASES + [CFG1]:
        recipe = build if isinstance(build, str) else ""
        A = build_recipe(build) if recipe else build()
        f = _run_reference(rq, driver, A, k, block, padding, seed)
        _store(name, driver, A, k, block, padding, seed, full, f, recipe)
        extra = "" if driver == "tuxv" else f" resamples={f.counters.resamples}"
        print(f"{name}: rank={f.rank}{extra}")


if __name__ == "__main__":
    if sys.argv[1:] in (["qr"], ["harness"], ["matio"]):   # one fixture only
        sys.path.insert(0, REF)
        import rqrcp as _rq
        {"qr": make_qr, "harness": make_harness, "matio": make_matio}[sys.argv[1]](_rq)
    else:
        main()
