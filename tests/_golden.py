"""Helpers to read the reference-generated fixtures in tests/golden/."""

import glob
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def case_names(prefix=""):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz"))):
        name = os.path.basename(p)[:-4]
        if not name.startswith(("kat_", "big_")):
            out.append(name)
    return out


def recipe_of(rec):
    return str(rec["recipe"]) if "recipe" in rec else ""


def portable(rec):
    """True when A is bit-identical on any host (stored, or a seeded Gaussian)."""
    return "A" in rec or recipe_of(rec).startswith("gauss:")


def matrix_of(rec):
    """The case's input A (stored, or rebuilt from its seeded recipe)."""
    if "A" in rec:
        return np.array(rec["A"], dtype=np.float64)
    import sys
    sys.path.insert(0, GOLDEN)
    from make_golden import build_recipe
    return build_recipe(recipe_of(rec))


def k_of(rec):
    k = int(rec["k"])
    return None if k < 0 else k
