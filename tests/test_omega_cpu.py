"""Host Omega stream (rq_omega_fill, csrc/omega.cu) against numpy's
Philox(key=seed).standard_normal -- the generator the reference's RngState
wraps (pkg/src/rqrcp/rng.py:16-41).  CPU only: the library loads without a GPU."""

import numpy as np
import pytest

import paper_1509_06820_b200.rng as R
from paper_1509_06820_b200.rng import RngState, gaussian_matrix


@pytest.mark.parametrize("threads", [1, 2, 5, 16])
@pytest.mark.parametrize("seed", [0, 1, 2**64 + 3])
def test_stream_bit_identical(threads, seed, monkeypatch):
    monkeypatch.setattr(R, "THREADS", threads)
    n = 200_003
    ref = np.random.Generator(np.random.Philox(key=seed)).standard_normal(n + 40_000)
    r = RngState(seed)
    parts = [r.draw(n), r.draw(1), r.draw(39_999)]
    np.testing.assert_array_equal(np.concatenate(parts), ref)
    assert r.position == n + 40_000


@pytest.mark.parametrize("pos", [0, 1, 72 * 1000, 123_457])
def test_position_replay(pos):
    ref = np.random.Generator(np.random.Philox(key=0)).standard_normal(pos + 5000)
    np.testing.assert_array_equal(RngState(0, position=pos).draw(5000), ref[pos:])


def test_column_major_kat():
    om = gaussian_matrix(RngState(0), 72, 1000)
    assert om[0, 0] == 0.15929546600623282 and om[1, 0] == -1.7741885208017214


def test_fill_rejects_bad_buffers():
    with pytest.raises(ValueError):
        RngState(0).fill(np.empty((4, 4))[:, ::2])
    with pytest.raises(ValueError):
        RngState(-1)
