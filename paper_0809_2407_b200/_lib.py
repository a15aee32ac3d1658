"""ctypes binding of libcaqr_sm100.so (the C-ABI declared in include/caqr_sm100.h).

The product path has no CPU fallback: if the library is missing or cannot be
loaded, every compute entry point raises ``NativeLibraryError``.  The library
is built in-tree by ``paper_0809_2407_b200.build`` / ``__graft_entry__.build()``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CAQR_SM100_LIB") or os.path.join(_HERE, "lib", "libcaqr_sm100.so")
ABI_VERSION = 1

# exported symbols, in header order (tests check each one is present)
SYMBOLS = (
    "caqr_sm100_abi_version",
    "tsqr_last_error",
    "tsqr_f64_geometry",
    "tsqr_f64_leaf_factor",
    "tsqr_f64_r_binary",
    "tsqr_f64_r_binary_rows",
    "tsqr_f64_r_combine_level",
    "tsqr_f64_colmajor_to_rowmajor",
    "tsqr_f64_tree_factor_level",
    "tsqr_f64_tree_apply_level",
    "tsqr_f64_leaf_apply",
    "tsqr_f64_leaf_factor_t",
    "tsqr_f64_leaf_apply_t",
    "tsqr_f64_panel_t_used",
    "tsqr_f64_block_factor",
    "tsqr_f64_block_apply",
    "tsqr_f64_geqr2",
    "tsqr_f64_form_t",
    "tsqr_f64_cholesky",
    "caqr_tune",
    "caqr_f64_peak_probe",
)

OK, ERR_ARG, ERR_NONFINITE, ERR_CUDA, ERR_COMM = 0, 1, 2, 3, 4


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing or failed to load (no CPU fallback)."""


_lib = None


def _sig(lib):
    i64, i32, vp, dp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p
    ip = ctypes.c_void_p
    lib.caqr_sm100_abi_version.restype = i32
    lib.caqr_sm100_abi_version.argtypes = []
    lib.tsqr_last_error.restype = ctypes.c_char_p
    lib.tsqr_last_error.argtypes = []
    lib.tsqr_f64_geometry.restype = i32
    lib.tsqr_f64_geometry.argtypes = [i64, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                      ctypes.POINTER(i64)]
    lib.tsqr_f64_panel_t_used.restype = i32
    lib.tsqr_f64_panel_t_used.argtypes = [i64]
    lib.tsqr_f64_leaf_factor_t.restype = i32
    lib.tsqr_f64_leaf_factor_t.argtypes = [dp, i64, i64, i64, i64, dp, i64, dp, i64, dp, ip, dp, vp]
    lib.tsqr_f64_leaf_apply_t.restype = i32
    lib.tsqr_f64_leaf_apply_t.argtypes = [dp, i64, dp, i64, i64, i64, i64, dp, i64, i64, dp, vp]
    lib.tsqr_f64_leaf_factor.restype = i32
    lib.tsqr_f64_leaf_factor.argtypes = [dp, i64, i64, i64, i64, dp, i64, dp, i64, dp, ip, vp]
    lib.tsqr_f64_r_binary.restype = i32
    lib.tsqr_f64_r_binary.argtypes = [dp, i64, i64, i64, i64, dp, ip, ip, vp]
    lib.tsqr_f64_r_binary_rows.restype = i32
    lib.tsqr_f64_r_binary_rows.argtypes = [dp, i64, i64, i64, i64, i64, dp, ip, ip, vp]
    lib.tsqr_f64_r_combine_level.restype = i32
    lib.tsqr_f64_r_combine_level.argtypes = [dp, i64, ip, i64, vp]
    lib.tsqr_f64_colmajor_to_rowmajor.restype = i32
    lib.tsqr_f64_colmajor_to_rowmajor.argtypes = [dp, i64, i64, i64, dp, i64, vp]
    lib.tsqr_f64_tree_factor_level.restype = i32
    lib.tsqr_f64_tree_factor_level.argtypes = [dp, i64, ip, i64, dp, dp, vp]
    lib.tsqr_f64_tree_apply_level.restype = i32
    lib.tsqr_f64_tree_apply_level.argtypes = [dp, dp, i64, ip, i64, dp, i64, i64, i64, i32, i32, vp]
    lib.tsqr_f64_leaf_apply.restype = i32
    lib.tsqr_f64_leaf_apply.argtypes = [dp, i64, dp, i64, i64, i64, i64, dp, i64, i64, dp, i64,
                                        i64, i32, i32, i32, vp]
    lib.tsqr_f64_block_factor.restype = i32
    lib.tsqr_f64_block_factor.argtypes = [dp, i64, i64, i64, dp, dp, i64, dp, i32, ip, vp]
    lib.tsqr_f64_block_apply.restype = i32
    lib.tsqr_f64_block_apply.argtypes = [dp, i64, i64, i64, dp, dp, i64, dp, i64, i64, i32, i32, vp]
    lib.tsqr_f64_geqr2.restype = i32
    lib.tsqr_f64_geqr2.argtypes = [dp, i64, i64, i64, dp, ip, vp]
    lib.tsqr_f64_form_t.restype = i32
    lib.tsqr_f64_form_t.argtypes = [dp, i64, i64, dp, dp, i64, vp]
    lib.tsqr_f64_cholesky.restype = i32
    lib.tsqr_f64_cholesky.argtypes = [dp, i64, i64, ip, vp]
    lib.caqr_tune.restype = i32
    lib.caqr_tune.argtypes = [i32, i32]
    lib.caqr_f64_peak_probe.restype = i32
    lib.caqr_f64_peak_probe.argtypes = [dp, i32, i32, i32, vp]


def load():
    """Load (once) and return the native library; raise if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - environment specific
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    missing = [s for s in SYMBOLS if not hasattr(lib, s)]
    if missing:
        raise NativeLibraryError(f"{LIB_PATH} lacks symbols {missing}")
    _sig(lib)
    if lib.caqr_sm100_abi_version() != ABI_VERSION:
        raise NativeLibraryError("ABI version mismatch; rebuild the library")
    _lib = lib
    # CAQR_TUNE="key=value,..." (caqr_tune keys, e.g. "12=0"): A/B runs of unmodified scripts
    for item in filter(None, os.environ.get("CAQR_TUNE", "").split(",")):
        k, v = item.split("=")
        check(lib.caqr_tune(int(k), int(v)), "CAQR_TUNE")
        TUNE_DEFAULTS[int(k)] = int(v)
    return lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI status code to the reference's exception types."""
    if rc == OK:
        return
    msg = (_lib.tsqr_last_error() or b"").decode(errors="replace")
    from .core import DimensionError
    from .executor import ExecutorError

    if rc == ERR_ARG:
        raise DimensionError(f"{what}: {msg}")
    if rc == ERR_NONFINITE:
        raise ValueError(f"{what}: matrix contains NaN or Inf entries")
    raise ExecutorError(f"{what}: {msg} (status {rc})")


TUNE_CHAIN_HT = {32: 1, 64: 2, 128: 3}
TUNE_NARROW = 4
TUNE_ZSTART = 6
TUNE_DMMA = 9
TUNE_DMMA_APPLY = 10
TUNE_DMMA_Q = 11
TUNE_DMMA_TREE = 12
TUNE_DMMA_TREE_FACTOR = 13
TUNE_DMMA_DENSE = 14
TUNE_CC = 15
TUNE_FUSE = 16
TUNE_NARROW_PF = 17


# the library's defaults (csrc/tsqr_sm100.cu, g_ht / g_narrow / ... initialisers)
TUNE_DEFAULTS = {TUNE_CHAIN_HT[32]: 16, TUNE_CHAIN_HT[64]: 16, TUNE_CHAIN_HT[128]: 16,
                 TUNE_NARROW: 3, TUNE_ZSTART: 1, TUNE_DMMA: 2,
                 TUNE_DMMA_APPLY: 1, TUNE_DMMA_Q: 1, TUNE_DMMA_TREE: 2,
                 TUNE_DMMA_TREE_FACTOR: 1, TUNE_DMMA_DENSE: 0, TUNE_CC: 5, TUNE_FUSE: 148, TUNE_NARROW_PF: 1}


def tune(key: int, value: int) -> None:
    check(load().caqr_tune(key, value), "caqr_tune")


def reset_tuning() -> None:
    """Restore every tuning knob to the library default."""
    for key, value in TUNE_DEFAULTS.items():
        tune(key, value)


def geometry(n: int):
    lib = load()
    np_, h0, ht = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    check(lib.tsqr_f64_geometry(n, ctypes.byref(np_), ctypes.byref(h0), ctypes.byref(ht)),
          "tsqr_f64_geometry")
    return np_.value, h0.value, ht.value
