"""Audit of the select kernel's 48-bit argmax key on the BASELINE inputs:
runs the oracle (bit-identical to the reference) with its argmax wrapped by
tests/test_argmax_key_cpu.KeyAudit and records how many pivot steps fall
inside the key's 2^-36 relative band, and the smallest relative gap between
the chosen norm and the best different norm.
Usage: python tools/argmax_band.py out.json cfg2 cfg3"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import recipes  # noqa: E402

from oracle import port  # noqa: E402
from tests.test_argmax_key_cpu import KeyAudit  # noqa: E402

out = {}
for name in sys.argv[2:]:
    drv, k, b, p, _ = recipes.CONFIGS[name]
    A = recipes.build(name)
    with KeyAudit() as audit:
        getattr(port, drv)(A, k, b, p, 0)
    out[name] = {"steps": audit.steps, "steps_inside_band": audit.mismatch,
                 "min_relative_gap": audit.min_gap, "band": 2.0 ** -36}
    print(name, out[name], flush=True)
json.dump(out, open(sys.argv[1], "w"), indent=1)
