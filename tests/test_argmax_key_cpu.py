"""The pivot selection (csrc/select.cu) orders candidates by a packed 64-bit
key: the top 48 bits of the downdated norm's IEEE pattern, then the
complemented 16-bit position.  Two norms that agree in those 48 bits (a
relative band of 2^-36, about 1.5e-11) are therefore ordered by position,
not by value.  This checks, on the reference's own norms (the oracle is
bit-identical to the reference, tests/test_oracle_golden.py), that no pivot
step of the fixtures falls inside that band, i.e. that the key's choice is
the reference's np.argmax choice at every step."""

import numpy as np
import pytest

from oracle import port
from tests import _golden as G


def key_of(v, pos):
    bits = np.asarray(v, dtype=np.float64).view(np.uint64) >> np.uint64(16)
    return (bits << np.uint64(16)) | np.uint64(0xFFFF) - np.asarray(pos, dtype=np.uint64)


class KeyAudit:
    """Wraps port.Norms.argmax_from: records where the 48-bit key would pick a
    different column than np.argmax, and the smallest relative gap between
    the winner and the best column of a different norm."""

    def __init__(self):
        self.mismatch = 0
        self.steps = 0
        self.min_gap = np.inf

    def __enter__(self):
        self.orig = port.Norms.argmax_from
        audit = self

        def argmax_from(tr, s):
            p, best = audit.orig(tr, s)
            vals = tr.val[s:]
            if vals.size > 1 and best > 0:
                audit.steps += 1
                pos = np.arange(vals.size)
                kp = int(np.argmax(key_of(vals, pos))) + s
                if kp != p:
                    audit.mismatch += 1
                other = vals[vals != best]
                if other.size:
                    audit.min_gap = min(audit.min_gap, float((best - other.max()) / best))
            return p, best

        port.Norms.argmax_from = argmax_from
        return self

    def __exit__(self, *exc):
        port.Norms.argmax_from = self.orig


def test_key_matches_exact_order_on_ties_and_near_ties():
    # exact ties keep the first position; a 2^-40 gap is inside the band
    v = np.array([1.0, 1.0, 0.5])
    assert int(np.argmax(key_of(v, np.arange(3)))) == 0
    w = np.array([1.0, 1.0 + 2.0 ** -40])
    assert int(np.argmax(key_of(w, np.arange(2)))) == 0   # np.argmax says 1: the band


@pytest.mark.parametrize("name", [n for n in G.case_names() if n.startswith(("rq_", "rs_", "ss_", "tr_", "cfg1"))])
def test_no_fixture_step_inside_the_key_band(name):
    rec = G.load(name)
    A = G.matrix_of(rec)
    k = G.k_of(rec)
    b, p, seed = int(rec["block"]), int(rec["padding"]), int(rec["seed"])
    drv = {"rqrcp": port.rqrcp, "rsrqrcp": port.rsrqrcp, "ssrqrcp": port.ssrqrcp,
           "trqrcp": port.trqrcp}[str(rec["driver"])]
    with KeyAudit() as audit:
        drv(A, k, b, p, seed)
    assert audit.mismatch == 0, f"{audit.mismatch} of {audit.steps} steps inside the 2^-36 band"
