"""The BASELINE configurations' input matrices, exactly as SURVEY.md §8(d)
writes them (numpy PCG64 + OpenBLAS LAPACK on the host), shared by the
golden generator (make_big_golden.py, which runs the reference) and the
full-size GPU parity tests (tests/test_gpu_fullsize.py).  The Gaussian-only
recipes (cfg1, cfg5) are bit-portable; the others go through LAPACK QR /
BLAS GEMM and are bit-stable only on hosts whose OpenBLAS picks the same
kernels, which is why every golden stores the sha256 of its A."""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
import tempfile

import numpy as np

# the OpenBLAS kernel family and thread count the goldens were generated with
# (threadpoolctl in the build container: architecture SkylakeX, 8 threads)
GOLDEN_BLAS = {"OPENBLAS_CORETYPE": "SkylakeX", "OPENBLAS_NUM_THREADS": "8"}

# name -> (driver, k, block, padding, description)
CONFIGS = {
    "cfg1": ("rqrcp", None, 32, 8, "1000x1000 Gaussian"),
    "cfg2": ("rqrcp", None, 64, 8, "8192x8192, sigma_i = 10^(-12 i / 8191)"),
    "cfg3": ("trqrcp", 512, 64, 8, "16384x16384 rank-600 Gaussian product + 1e-6 noise"),
    "cfg4": ("tuxv", 256, 32, 8, "20000x12000, sigma_i = 1/(1+i)^2"),
    "cfg5": ("rqrcp", None, 128, 8, "32768x32768 Gaussian"),
}


def sha(a) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def build(name: str) -> np.ndarray:
    """F-ordered float64 input of configuration `name`."""
    if name == "cfg1":
        return np.asfortranarray(np.random.default_rng(0).standard_normal((1000, 1000)))
    if name == "cfg2":
        rng = np.random.default_rng(0)
        U = np.linalg.qr(rng.standard_normal((8192, 8192)))[0]
        V = np.linalg.qr(rng.standard_normal((8192, 8192)))[0]
        s = 10.0 ** (-12.0 * np.arange(8192) / 8191)
        return np.asfortranarray((U * s) @ V.T)
    if name == "cfg3":
        rng = np.random.default_rng(0)
        G1 = rng.standard_normal((16384, 600))
        G2 = rng.standard_normal((600, 16384))
        A = G1 @ G2
        A += 1e-6 * rng.standard_normal((16384, 16384))
        return np.asfortranarray(A)
    if name == "cfg4":
        rng = np.random.default_rng(0)
        U = np.linalg.qr(rng.standard_normal((20000, 12000)))[0]
        V = np.linalg.qr(rng.standard_normal((12000, 12000)))[0]
        s = 1.0 / (1.0 + np.arange(12000)) ** 2
        return np.asfortranarray((U * s) @ V.T)
    if name == "cfg5":
        return np.asfortranarray(np.random.default_rng(0).standard_normal((32768, 32768)))
    raise KeyError(name)


def _avx512():
    try:
        return " avx512f" in open("/proc/cpuinfo").read()
    except OSError:
        return False


def build_as_golden(name: str) -> np.ndarray:
    """build(name) in a subprocess whose OpenBLAS uses the golden host's
    kernel family and thread count, so LAPACK-built recipes reproduce the
    golden's bytes on another host (the kernel choice is made when the
    library loads, hence the fresh process).  Falls back to build() when the
    CPU cannot run those kernels."""
    if name in ("cfg1", "cfg5") or not _avx512():
        return build(name)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "A.npy")
        env = dict(os.environ, **GOLDEN_BLAS)
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import recipes; "
                "np.save(%r, recipes.build(%r))" % (os.path.dirname(os.path.abspath(__file__)),
                                                    out, name))
        subprocess.run([sys.executable, "-c", code], check=True, env=env)
        return np.asfortranarray(np.load(out))
