"""B200-native FP64 TSQR / CAQR (arXiv:0809.2407) -- the hot path of the
reference ``caqr`` package re-built on hand-written sm_100a kernels.

Public API (reference names):
    tsqr.tsqr, tsqr_parallel, tsqr_explicit_q, tsqr_apply_q, TsqrFactor
    caqr_factor, gather_R, caqr_apply_q, CaqrResult
plus the reference's host utilities (core, trees, counters) and the
executor plugin point (DeviceExecutor).
"""

from .core import (  # noqa: F401
    BlockCyclicLayout,
    BlockRowLayout,
    CondSpec,
    DimensionError,
    as_matrix,
    gen_cond_matrix,
    partition_block_rows,
    rng_for,
)
from .executor import DeviceExecutor, ExecutorError, LocalExecutor, Message, payload_words  # noqa: F401
from .trees import ReductionTree, TreeError, parse_tree  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):  # lazy: the compute modules need torch + the CUDA library
    if name in ("tsqr_parallel", "tsqr_explicit_q", "tsqr_apply_q", "TsqrFactor"):
        from . import tsqr as _t

        return getattr(_t, name)
    if name in ("caqr_factor", "gather_R", "caqr_apply_q", "CaqrResult"):
        from . import caqr as _c

        return getattr(_c, name)
    raise AttributeError(name)
