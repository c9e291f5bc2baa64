"""numpy restatement of the reference's randomized pivoted QR (test oracle).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  The product package
never imports this module.

Every floating-point operation below is the same numpy call the reference
makes, in the same order, so on the same numpy/OpenBLAS build the outputs are
bitwise identical to the reference (``tests/test_oracle_golden.py`` pins that
against fixtures generated from /root/reference).  The code is organised
differently from the reference: one mutable ``_Run`` state object per driver
call instead of module-level helpers, and the three drivers share one block
loop.

Reference citations are ``pkg/src/rqrcp/<file>:<line>``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

EPS = float(np.finfo(np.float64).eps)
NORM_GUARD = float(np.sqrt(np.finfo(np.float64).eps))  # kernels.py:205


# --------------------------------------------------------------------------
# accounting, Ω stream


@dataclass
class Counters:
    """Mirror of OpCounters (counters.py:12-27)."""

    gemm_flops: int = 0
    level2_flops: int = 0
    bytes_touched: int = 0
    resamples: int = 0

    def touch(self, *arrays):
        for a in arrays:
            self.bytes_touched += 8 * int(np.size(a))


class Stream:
    """Seeded Philox standard-normal stream with a replayable position
    (rng.py:16-33); matrices are filled column-major (rng.py:36-41)."""

    def __init__(self, seed, position=0):
        self.seed = seed
        self.position = 0
        self._g = np.random.Generator(np.random.Philox(key=seed))
        if position:
            self._g.standard_normal(position)
            self.position = position

    def matrix(self, rows, cols):
        if rows < 1 or cols < 1:
            raise ValueError("gaussian_matrix needs rows, cols >= 1")
        flat = self._g.standard_normal(rows * cols)
        self.position += rows * cols
        return np.asfortranarray(flat.reshape((rows, cols), order="F"))


# --------------------------------------------------------------------------
# level-1/2 primitives (kernels.py)


def householder(x):
    """(v, tau, beta) with v[0] = 1 and beta = -sign(x0)*||x||, sign(0)=+1;
    the zero vector gives tau = beta = 0 (kernels.py:26-44)."""
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise ValueError("form_reflector needs a nonempty vector")
    v = x.copy()
    nrm = float(np.linalg.norm(x))
    if nrm == 0.0:
        v[0] = 1.0
        return v, 0.0, 0.0
    a0 = float(x[0])
    beta = nrm if a0 < 0.0 else -nrm
    v /= a0 - beta
    v[0] = 1.0
    return v, (beta - a0) / beta, beta


def reflect_left(M, v, tau, ctr=None):
    """M <- (I - tau v v^T) M in place (kernels.py:47-56)."""
    if M.shape[1] == 0 or tau == 0.0:
        return M
    w = v @ M
    M -= np.outer(tau * v, w)
    if ctr is not None:
        ctr.level2_flops += 4 * M.shape[0] * M.shape[1]
        ctr.touch(M, M)
    return M


def t_factor(Y, tau):
    """Forward column-wise T with I - Y T Y^T = H_1...H_b (kernels.py:139-147)."""
    nb = Y.shape[1]
    T = np.zeros((nb, nb))
    for j in range(nb):
        T[j, j] = tau[j]
        if j:
            T[:j, j] = -tau[j] * (T[:j, :j] @ (Y[:, :j].T @ Y[:, j]))
    return T


class Perm:
    """forward map + ordered swap log (kernels.py:59-111)."""

    def __init__(self, n):
        self.forward = np.arange(n)
        self.swaps = []

    def swap(self, i, j):
        self.swaps.append((i, j))
        if i != j:
            self.forward[[i, j]] = self.forward[[j, i]]

    def restore(self, R):
        out = np.zeros_like(R)
        out[:, self.forward] = R
        return out


class Norms:
    """Downdated trailing column norms with the sqrt(eps) recompute guard
    (kernels.py:196-233)."""

    def __init__(self, M):
        self.val = np.linalg.norm(M, axis=0)
        self.ref_sq = self.val**2

    def swap(self, i, j):
        if i != j:
            self.val[[i, j]] = self.val[[j, i]]
            self.ref_sq[[i, j]] = self.ref_sq[[j, i]]

    def argmax_from(self, s):
        p = int(np.argmax(self.val[s:])) + s
        return p, self.val[p]

    def downdate(self, s, row, column_of):
        sq = self.val[s:] ** 2 - np.asarray(row) ** 2
        np.maximum(sq, 0.0, out=sq)
        bad = sq < NORM_GUARD * self.ref_sq[s:]
        self.val[s:] = np.sqrt(sq)
        for off in np.nonzero(bad)[0]:
            c = s + int(off)
            fresh = float(np.linalg.norm(column_of(c)))
            self.val[c] = fresh
            self.ref_sq[c] = fresh * fresh


def greedy_eliminate(M, steps, Y, tau, perm, tol, ctr):
    """Greedy max-norm pivoted Householder steps on M in place; returns the
    steps completed (qrcp.py:63-84)."""
    ncol = M.shape[1]
    tr = Norms(M)
    for j in range(steps):
        p, best = tr.argmax_from(j)
        if best <= tol:
            return j
        if p != j:
            M[:, [j, p]] = M[:, [p, j]]
        perm.swap(j, p)
        tr.swap(j, p)
        v, t, beta = householder(M[j:, j])
        Y[j:, j] = v
        tau[j] = t
        reflect_left(M[j:, j + 1 :], v, t, ctr)
        M[j, j] = beta
        M[j + 1 :, j] = 0.0
        if j + 1 < ncol:
            tr.downdate(j + 1, M[j, j + 1 :], lambda c: M[j + 1 :, c])
    return steps


def panel_qr(P, ctr=None):
    """Unpivoted Householder QR of a panel copy in place (qrcp.py:206-219)."""
    rows, cols = P.shape
    Y = np.zeros((rows, cols))
    tau = np.zeros(cols)
    for j in range(min(rows, cols)):
        v, t, beta = householder(P[j:, j])
        Y[j:, j] = v
        tau[j] = t
        reflect_left(P[j:, j + 1 :], v, t, ctr)
        P[j, j] = beta
        P[j + 1 :, j] = 0.0
    return Y, tau


def q_columns(Y, tau, cols):
    """Leading columns of I - Y T Y^T (qrcp.py:53-60)."""
    Q = np.eye(Y.shape[0], cols)
    if Y.shape[1]:
        T = t_factor(Y, tau)
        Q -= Y @ (T @ (Y.T @ Q))
    return Q


def check_rank(k, m, n):
    """qrcp.py:87-94."""
    top = min(m, n)
    if k is None:
        return top
    k = int(k)
    if not 0 <= k <= top:
        raise ValueError(f"rank {k} outside [0, {top}]")
    return k


# --------------------------------------------------------------------------
# sample handling (randomized.py:48-135)


class Degenerate(RuntimeError):
    """randomized.py:43-45."""


@dataclass
class Sample:
    B: np.ndarray
    ell: int
    frob_a: float = 0.0
    s11: np.ndarray | None = None
    s12: np.ndarray | None = None
    s22: np.ndarray | None = None
    Ys: np.ndarray | None = None
    taus: np.ndarray | None = None


def sketch(M, ell, stream, ctr):
    """B = Omega M with a fresh ell x rows Omega (randomized.py:69-82)."""
    M = np.asarray(M, dtype=np.float64)
    if ell < 1:
        raise ValueError("sample must have at least one row")
    om = stream.matrix(ell, M.shape[0])
    B = om @ M
    if ctr is not None:
        ctr.gemm_flops += 2 * ell * M.shape[0] * M.shape[1]
        ctr.touch(om, M, B)
    return Sample(B=np.asfortranarray(B), ell=ell, frob_a=float(np.linalg.norm(M)))


def pick_pivots(smp, want, ctr):
    """want greedy steps on the sample in place (randomized.py:85-104)."""
    B = smp.B
    ell, nt = B.shape
    if not 1 <= want <= min(ell, nt):
        raise ValueError(f"cannot select {want} pivots from a {ell} x {nt} sample")
    perm = Perm(nt)
    Ys = np.zeros((ell, want))
    taus = np.zeros(want)
    tol = EPS * float(np.linalg.norm(B))
    got = greedy_eliminate(B, want, Ys, taus, perm, tol, ctr)
    smp.Ys, smp.taus = Ys[:, :got], taus[:got]
    smp.s11, smp.s12, smp.s22 = B[:got, :got], B[:got, got:], B[got:, got:]
    return perm, got


def downdate_sample(smp, R11, R12, ctr):
    """B <- [S12 - S11 R11^{-1} R12; S22] with the eps^(3/4) guard
    (randomized.py:107-135)."""
    nb = R11.shape[0]
    if smp.s11 is None or smp.s11.shape[0] != nb:
        raise ValueError("sample has no matching factorization to downdate")
    if np.any(np.abs(np.diag(R11)) < EPS**0.75 * smp.frob_a):
        raise Degenerate("block triangle numerically singular")
    n2 = R12.shape[1]
    if n2:
        X = np.linalg.solve(R11, R12)
        top = smp.s12 - smp.s11 @ X
        ctr.gemm_flops += 3 * nb * nb * n2
        ctr.touch(R11, R12, smp.s11, smp.s12, top)
        nxt = np.vstack([top, smp.s22])
    else:
        nxt = np.zeros((smp.ell, 0))
    smp.B = np.asfortranarray(nxt)
    smp.s11 = smp.s12 = smp.s22 = smp.Ys = smp.taus = None
    return smp


def replay_swaps(local, i0, perm, work, *followers):
    """randomized.py:138-147."""
    for a, c in local.swaps:
        ga, gc = i0 + a, i0 + c
        perm.swap(ga, gc)
        if ga != gc:
            work[:, [ga, gc]] = work[:, [gc, ga]]
            for F in followers:
                F[[ga, gc], :] = F[[gc, ga], :]


def usable_columns(R, tol):
    """randomized.py:150-155."""
    d = np.abs(np.diag(R))
    bad = d <= tol
    return int(np.argmax(bad)) if bad.any() else d.size


# --------------------------------------------------------------------------
# results


@dataclass
class Result:
    Y: np.ndarray
    tau: np.ndarray
    R: np.ndarray
    perm: Perm
    rank: int
    counters: Counters
    trailing: np.ndarray | None = None
    W: np.ndarray | None = None
    # oracle-only diagnostics: (i0, trigger) for every resample
    events: list = field(default_factory=list)

    def q_factor(self, full=False):
        return q_columns(self.Y, self.tau, self.Y.shape[0] if full else self.rank)


@dataclass
class TuxvResult:
    U: np.ndarray
    V: np.ndarray
    X: np.ndarray
    iterations: int
    rank: int
    counters: Counters

    def approx(self):
        return self.U @ (self.X @ self.V.T)

    def singular_values(self):
        return np.sort(np.abs(np.diag(self.X)))[::-1]


# --------------------------------------------------------------------------
# RQRCP family (randomized.py:158-313)


def _push_block(work, Yb, tb, i0, bw, ctr, update_trailing):
    """X = T^T (Y^T C); R12 = C[:b] - Y[:b] X; optional C[b:] -= Y[b:] X
    (randomized.py:158-180)."""
    m, n = work.shape
    nt2 = n - i0 - bw
    if not nt2:
        return
    T = t_factor(Yb, tb)
    C = work[i0:, i0 + bw :]
    X = T.T @ (Yb.T @ C)
    ctr.gemm_flops += 2 * (m - i0) * bw * nt2 + bw * bw * nt2
    work[i0 : i0 + bw, i0 + bw :] = C[:bw] - Yb[:bw] @ X
    ctr.gemm_flops += 2 * bw * bw * nt2
    ctr.touch(C, Yb, X)
    if update_trailing and i0 + bw < m:
        work[i0 + bw :, i0 + bw :] = C[bw:] - Yb[bw:] @ X
        ctr.gemm_flops += 2 * (m - i0 - bw) * bw * nt2
        ctr.touch(work[i0 + bw :, i0 + bw :])


def randomized_factor(A, k, seed, ell, width, resketch_each_block, update_trailing,
                      omega0=None):
    """Shared block loop of rqrcp / rsrqrcp / ssrqrcp
    (randomized.py:183-266).  ``omega0`` optionally replaces the first
    ell x m draw (the stream then continues at position ell*m)."""
    work = np.array(A, dtype=np.float64, order="F")
    m, n = work.shape
    k = check_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    if ell > m:
        raise ValueError(f"sample rows {ell} exceed matrix rows {m}")
    stream = Stream(seed)
    ctr = Counters()
    frob = float(np.linalg.norm(work))
    tol = EPS * frob
    perm = Perm(n)
    Y = np.zeros((m, k))
    tau = np.zeros(k)
    events = []

    def resketch(i0):
        s = sketch(work[i0:, i0:], ell, stream, ctr)
        s.frob_a = frob
        return s

    if omega0 is not None:
        stream = Stream(seed, position=ell * m)
        om = np.asfortranarray(np.asarray(omega0, dtype=np.float64))
        smp = Sample(B=np.asfortranarray(om @ work), ell=ell, frob_a=frob)
        ctr.gemm_flops += 2 * ell * m * n
        ctr.touch(om, work, smp.B)
    else:
        smp = resketch(0)
    rank = k
    i0 = 0
    while i0 < k:
        want = min(width, k - i0)
        again = False
        while True:
            local, got = pick_pivots(smp, want, ctr)
            if got < want and not again:
                smp = resketch(i0)
                ctr.resamples += 1
                events.append((i0, "short_sample"))
                again = True
                continue
            if got == 0:
                bw = 0
                break
            replay_swaps(local, i0, perm, work)
            P = work[i0:, i0 : i0 + got].copy()
            Yp, tp = panel_qr(P, ctr)
            ok = usable_columns(P, tol)
            if ok < got and not again:
                smp = resketch(i0)
                ctr.resamples += 1
                events.append((i0, "panel_rank"))
                again = True
                continue
            bw = ok
            if bw:
                work[i0:, i0 : i0 + bw] = P[:, :bw]
                Y[i0:, i0 : i0 + bw] = Yp[:, :bw]
                tau[i0 : i0 + bw] = tp[:bw]
            break
        if bw == 0:
            rank = i0
            break
        _push_block(work, Y[i0:, i0 : i0 + bw], tau[i0 : i0 + bw], i0, bw, ctr,
                    update_trailing)
        i0 += bw
        if bw < want:
            rank = i0
            break
        if i0 < k:
            if resketch_each_block:
                smp = resketch(i0)
            else:
                try:
                    downdate_sample(smp, work[i0 - bw : i0, i0 - bw : i0],
                                    work[i0 - bw : i0, i0:], ctr)
                except Degenerate:
                    smp = resketch(i0)
                    ctr.resamples += 1
                    events.append((i0, "degenerate"))
    return Result(
        Y=Y[:, :rank], tau=tau[:rank], R=work[:rank, :].copy(), perm=perm, rank=rank,
        counters=ctr, trailing=work[rank:, rank:].copy() if update_trailing else None,
        events=events,
    )


def rqrcp(A, k=None, block=32, padding=8, seed=0, omega=None):
    """randomized.py:269-281."""
    return randomized_factor(A, k, seed, block + padding, block, False, True, omega)


def rsrqrcp(A, k=None, block=32, padding=8, seed=0, omega=None):
    """randomized.py:284-296."""
    return randomized_factor(A, k, seed, block + padding, block, True, True, omega)


def ssrqrcp(A, k, block=32, padding=8, seed=0, omega=None):
    """randomized.py:299-313."""
    k = int(k)
    return randomized_factor(A, k, seed, k + padding, k, False, False, omega)


# --------------------------------------------------------------------------
# TRQRCP / TUXV (truncated.py)


def _implicit_sketch(work, Y, W, i0, ell, stream, ctr, frob):
    """Sketch of the never-formed trailing matrix (truncated.py:53-67)."""
    m, n = work.shape
    om = stream.matrix(ell, m - i0)
    B = om @ work[i0:, i0:]
    ctr.gemm_flops += 2 * ell * (m - i0) * (n - i0)
    ctr.touch(om, work[i0:, i0:], B)
    if i0:
        B -= (om @ Y[i0:, :i0]) @ W[i0:, :i0].T
        ctr.gemm_flops += 2 * ell * (m - i0) * i0 + 2 * ell * i0 * (n - i0)
        ctr.touch(Y[i0:, :i0], W[i0:, :i0])
    return Sample(B=np.asfortranarray(B), ell=ell, frob_a=frob)


def trqrcp(A, k, block=32, padding=8, seed=0, omega=None):
    """Truncated RQRCP, no trailing update (truncated.py:70-174)."""
    work = np.array(A, dtype=np.float64, order="F")
    m, n = work.shape
    k = check_rank(k, m, n)
    if k == 0:
        raise ValueError("rank must be >= 1")
    ell = block + padding
    if ell > m:
        raise ValueError(f"sample rows {ell} exceed matrix rows {m}")
    stream = Stream(seed)
    ctr = Counters()
    frob = float(np.linalg.norm(work))
    tol = EPS * frob
    perm = Perm(n)
    Y = np.zeros((m, k))
    tau = np.zeros(k)
    W = np.zeros((n, k))
    R = np.zeros((k, n), order="F")
    events = []
    if omega is not None:
        stream = Stream(seed, position=ell * m)
        om = np.asfortranarray(np.asarray(omega, dtype=np.float64))
        smp = Sample(B=np.asfortranarray(om @ work), ell=ell, frob_a=frob)
        ctr.gemm_flops += 2 * ell * m * n
        ctr.touch(om, work, smp.B)
    else:
        smp = sketch(work, ell, stream, ctr)
        smp.frob_a = frob
    rank = k
    i0 = 0
    while i0 < k:
        want = min(block, k - i0)
        again = False
        while True:
            local, got = pick_pivots(smp, want, ctr)
            if got < want and not again:
                smp = _implicit_sketch(work, Y, W, i0, ell, stream, ctr, frob)
                ctr.resamples += 1
                events.append((i0, "short_sample"))
                again = True
                continue
            if got == 0:
                bw = 0
                break
            replay_swaps(local, i0, perm, work, W, R.T)
            P = work[i0:, i0 : i0 + got].copy()
            if i0:
                P -= Y[i0:, :i0] @ W[i0 : i0 + got, :i0].T
                ctr.gemm_flops += 2 * (m - i0) * i0 * got
                ctr.touch(P, Y[i0:, :i0], W[i0 : i0 + got, :i0])
            Yp, tp = panel_qr(P, ctr)
            ok = usable_columns(P, tol)
            if ok < got and not again:
                smp = _implicit_sketch(work, Y, W, i0, ell, stream, ctr, frob)
                ctr.resamples += 1
                events.append((i0, "panel_rank"))
                again = True
                continue
            bw = ok
            if bw:
                Y[i0:, i0 : i0 + bw] = Yp[:, :bw]
                tau[i0 : i0 + bw] = tp[:bw]
                R[i0 : i0 + bw, i0 : i0 + bw] = P[:bw, :bw]
            break
        if bw == 0:
            rank = i0
            break
        Yb = Y[i0:, i0 : i0 + bw]
        nt2 = n - i0 - bw
        if nt2:
            T = t_factor(Yb, tau[i0 : i0 + bw])
            G = Yb.T @ work[i0:, i0 + bw :]
            ctr.gemm_flops += 2 * (m - i0) * bw * nt2
            if i0:
                G -= (Yb.T @ Y[i0:, :i0]) @ W[i0 + bw :, :i0].T
                ctr.gemm_flops += 2 * (m - i0) * bw * i0 + 2 * bw * i0 * nt2
            W[i0 + bw :, i0 : i0 + bw] = (T.T @ G).T
            ctr.gemm_flops += bw * bw * nt2
            R[i0 : i0 + bw, i0 + bw :] = (
                work[i0 : i0 + bw, i0 + bw :]
                - Y[i0 : i0 + bw, : i0 + bw] @ W[i0 + bw :, : i0 + bw].T
            )
            ctr.gemm_flops += 2 * bw * (i0 + bw) * nt2
            ctr.touch(R[i0 : i0 + bw, :], W[i0 + bw :, : i0 + bw])
        i0 += bw
        if bw < want:
            rank = i0
            break
        if i0 < k:
            try:
                downdate_sample(smp, R[i0 - bw : i0, i0 - bw : i0], R[i0 - bw : i0, i0:], ctr)
            except Degenerate:
                smp = _implicit_sketch(work, Y, W, i0, ell, stream, ctr, frob)
                ctr.resamples += 1
                events.append((i0, "degenerate"))
    return Result(
        Y=Y[:, :rank], tau=tau[:rank], R=R[:rank, :].copy(), perm=perm, rank=rank,
        counters=ctr, W=W[:, :rank], events=events,
    )


def qr_blocked(A, k=None, b=32, ctr=None):
    """Unpivoted blocked QR (qrcp.py:222-252); returns (Y, tau, R)."""
    work = np.array(A, dtype=np.float64, order="F")
    m, n = work.shape
    k = check_rank(k, m, n)
    if b < 1:
        raise ValueError("block size must be >= 1")
    ctr = ctr if ctr is not None else Counters()
    Y = np.zeros((m, k))
    tau = np.zeros(k)
    for i0 in range(0, k, b):
        bw = min(b, k - i0)
        Yp, tp = panel_qr(work[i0:, i0 : i0 + bw], ctr)
        Y[i0:, i0 : i0 + bw] = Yp
        tau[i0 : i0 + bw] = tp
        if i0 + bw < n:
            T = t_factor(Yp, tp)
            C = work[i0:, i0 + bw :]
            # apply_block_reflection(transpose=True), kernels.py:166-181
            Wt = Yp.T @ C
            Wt = T.T @ Wt
            C -= Yp @ Wt
            ctr.gemm_flops += 4 * C.shape[0] * bw * C.shape[1] + bw * bw * C.shape[1]
            ctr.touch(C, Yp, Wt, C)
    return Y, tau, work[:k, :].copy()


def column_norms(A):
    """np.linalg.norm(A, axis=0) (kernels.py:184-186); the summation order
    follows A's memory layout, as numpy's does."""
    return np.linalg.norm(A, axis=0)


def qr_presorted(A, k=None, b=32, ctr=None):
    """Blocked QR after a stable descending sort of the initial column norms
    (qrcp.py:255-268); returns (Y, tau, R, order)."""
    A = np.asarray(A, dtype=np.float64)
    order = np.argsort(-column_norms(A), kind="stable")
    Y, tau, R = qr_blocked(A[:, order], k=k, b=b, ctr=ctr)
    return Y, tau, R, order


def lq_factor(Z, b=32, ctr=None):
    """Z = L V^T through QR of Z^T (truncated.py:177-184)."""
    Z = np.asarray(Z, dtype=np.float64)
    Y, tau, R = qr_blocked(Z.T, b=b, ctr=ctr)
    return R.T, q_columns(Y, tau, Y.shape[1])


def tuxv(A, k, block=32, padding=8, seed=0, j_max=1, omega=None):
    """QLP-style approximate truncated SVD (truncated.py:208-252); the
    svd_of_x rotation is not part of the oracle (it calls the reference's
    Jacobi SVD, which is out of scope)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    if j_max < 1:
        raise ValueError("j_max must be >= 1")
    tf = trqrcp(A, k, block, padding, seed, omega)
    ctr = tf.counters
    r = tf.rank
    Z = tf.perm.restore(tf.R)
    _, V = lq_factor(Z, b=block, ctr=ctr)
    j = 1
    while True:
        Zc = A @ V[:, :r]
        ctr.gemm_flops += 2 * m * n * r
        ctr.touch(A, V[:, :r], Zc)
        Yq, tq, Rq = qr_blocked(Zc, b=block, ctr=ctr)
        U = q_columns(Yq, tq, Yq.shape[1])
        X = Rq[:, :r]
        if j >= j_max:
            break
        Zr = U.T @ A
        ctr.gemm_flops += 2 * m * n * r
        ctr.touch(U, Zr)
        X, V = lq_factor(Zr, b=block, ctr=ctr)
        if j + 1 >= j_max:
            break
        j += 2
    return TuxvResult(U=U, V=V[:, :r], X=X, iterations=j_max, rank=r, counters=ctr)
