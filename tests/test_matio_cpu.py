"""On-disk formats (paper_1509_06820_b200/matio.py) against the reference's
matio.py:25-238 behaviour, recorded in tests/golden/kat_matio.npz by
tests/golden/make_golden.py: parsed matrices bit for bit, the same error
class and message for malformed files, byte-identical writers."""

import numpy as np
import pytest

from paper_1509_06820_b200 import matio as M
from tests import _golden as G

REC = G.load("kat_matio")
CASES = sorted({k.rsplit("_", 1)[0] for k in REC if k.endswith("_bytes")})


@pytest.mark.parametrize("name", CASES)
def test_loader_matches_reference(tmp_path, name):
    fn = tmp_path / name
    fn.write_bytes(REC[name + "_bytes"].tobytes())
    load = M.load_matrix_market if name.startswith("mm") else M.load_pgm
    if name + "_out" in REC:
        out = load(fn)
        np.testing.assert_array_equal(out, REC[name + "_out"])
        if name.startswith("mm"):
            assert out.flags.f_contiguous
    else:
        with pytest.raises(ValueError) as ei:
            load(fn)
        got = type(ei.value).__name__ + ": " + str(ei.value).replace(str(fn), "{path}")
        assert got == str(REC[name + "_err"])


def test_writers_match_reference(tmp_path):
    M.save_matrix_market(REC["save_A"], tmp_path / "a.mtx")
    assert (tmp_path / "a.mtx").read_bytes() == REC["save_mtx"].tobytes()
    np.testing.assert_array_equal(M.load_matrix_market(tmp_path / "a.mtx"), REC["save_A"])
    for asc in (0, 1):
        for mv in (255, 1000):
            fn = tmp_path / f"s{asc}{mv}.pgm"
            M.save_pgm(REC["save_img"], fn, mv, bool(asc))
            assert fn.read_bytes() == REC[f"save_pgm_{asc}_{mv}"].tobytes()


def test_writer_validation():
    with pytest.raises(ValueError):
        M.save_matrix_market(np.array([1.0, np.inf])[None], "/dev/null")
    with pytest.raises(ValueError):
        M.save_pgm(np.zeros((2, 2)), "/dev/null", maxval=0)
