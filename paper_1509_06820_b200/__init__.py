"""B200-native (sm_100a) blocked Randomized QR with Column Pivoting.

Drop-in for the hot path of the reference package ``rqrcp`` (arXiv
1509.06820): ``rqrcp``, ``rsrqrcp``, ``ssrqrcp``, ``trqrcp``, ``tuxv``,
``lq_factor``, ``RandomizedConfig`` and the result types keep the reference
signatures (plus an optional explicit ``omega``).  All arithmetic runs in
librqrcp_b200.so (FP64 DMMA tensor-core GEMMs, cooperative pivot-selection
and panel kernels, a native block-loop driver); PyTorch only allocates
device memory and provides streams.  There is no CPU fallback.
"""

from .factorization import (
    BlockReflectors,
    Factorization,
    OpCounters,
    Permutation,
    TruncatedFactorization,
    TuxvFactorization,
    q_columns,
    t_factor,
)
from .matio import (
    MatrixFormatError,
    PgmFormatError,
    load_matrix_market,
    load_pgm,
    save_matrix_market,
    save_pgm,
)
from .qrcp import column_norms, qr_blocked, qr_presorted
from .kernels import (
    NormTracker,
    Reflector,
    apply_block_reflection,
    apply_reflector,
    compose_blocks,
    downdate_norms,
    form_reflector,
)
from .randomized import (
    DegenerateSampleError,
    RandomizedConfig,
    SampleState,
    make_sample,
    rqrcp,
    rsrqrcp,
    sample_update,
    select_pivots,
    ssrqrcp,
)
from .rng import RngState, gaussian_matrix
from .truncated import lq_factor, qr_blocked_device, trqrcp, tuxv

build_t_matrix = t_factor

__version__ = "0.1.0"

__all__ = [
    "BlockReflectors",
    "DegenerateSampleError",
    "NormTracker",
    "Reflector",
    "SampleState",
    "apply_block_reflection",
    "apply_reflector",
    "compose_blocks",
    "downdate_norms",
    "form_reflector",
    "make_sample",
    "sample_update",
    "select_pivots",
    "Factorization",
    "MatrixFormatError",
    "OpCounters",
    "PgmFormatError",
    "Permutation",
    "RandomizedConfig",
    "RngState",
    "TruncatedFactorization",
    "TuxvFactorization",
    "build_t_matrix",
    "column_norms",
    "gaussian_matrix",
    "load_matrix_market",
    "load_pgm",
    "lq_factor",
    "q_columns",
    "qr_blocked",
    "qr_blocked_device",
    "qr_presorted",
    "rqrcp",
    "rsrqrcp",
    "save_matrix_market",
    "save_pgm",
    "ssrqrcp",
    "t_factor",
    "trqrcp",
    "tuxv",
    "__version__",
]
