"""Matrix files: the reference's MAT1 / CSV interchange
(pkg/src/caqr/matio.py:1-74) and TSQR straight from a MAT1 file.

MAT1 (little-endian): 8-byte magic ``TSQRMAT1``, u32 rows, u32 cols, two
reserved u32 (24-byte header), then rows*cols float64 in COLUMN-major order
(matio.py:3-10).  The kernels read rows, so ``tsqr_mat1`` memory-maps the
file, stages each row chunk as n column segments in pinned memory and
transposes it on the GPU while the previous chunk is factored
(``stream.tsqr_stream``, ``tsqr_f64_colmajor_to_rowmajor``): the file is read
once, never materialised whole in host or device memory.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .core import as_matrix

MAGIC = b"TSQRMAT1"
_HEAD = struct.Struct("<8sIIII")  # magic, rows, cols, 2 x reserved (matio.py:22)
HEADER = _HEAD  # the reference's public name (tests build headers with it)


class FormatError(ValueError):
    """Malformed MAT1 file (matio.py:25-26)."""


def _header(path):
    with open(path, "rb") as f:
        head = f.read(_HEAD.size)
    if len(head) != _HEAD.size:
        raise FormatError(f"{path}: truncated header")
    magic, rows, cols, _, _ = _HEAD.unpack(head)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    size = Path(path).stat().st_size
    if size < _HEAD.size + 8 * rows * cols:
        raise FormatError(f"{path}: expected {rows}x{cols} doubles, file too short")
    return rows, cols


def write_mat1(path, A) -> None:
    """matio.py:29-34."""
    A = as_matrix(A)
    rows, cols = A.shape
    with open(path, "wb") as f:
        f.write(_HEAD.pack(MAGIC, rows, cols, 0, 0))
        f.write(np.asarray(A, dtype="<f8").tobytes(order="F"))


def open_mat1(path) -> np.ndarray:
    """Read-only column-major (Fortran-ordered) memory map of a MAT1 matrix."""
    rows, cols = _header(path)
    return np.memmap(path, dtype="<f8", mode="r", offset=_HEAD.size, shape=(rows, cols), order="F")


def read_mat1(path) -> np.ndarray:
    """matio.py:37-51: the whole matrix, C-ordered float64, NaN/Inf rejected."""
    return as_matrix(np.array(open_mat1(path), order="C"), str(path))


def write_csv(path, A) -> None:
    np.savetxt(path, as_matrix(A), delimiter=",", fmt="%.17g")


def read_csv(path) -> np.ndarray:
    return as_matrix(np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2), str(path))


def read_matrix(path) -> np.ndarray:
    """Dispatch on extension: .csv -> CSV, else MAT1 (matio.py:62-67)."""
    return read_csv(path) if Path(path).suffix.lower() == ".csv" else read_mat1(path)


def write_matrix(path, A) -> None:
    if Path(path).suffix.lower() == ".csv":
        write_csv(path, A)
    else:
        write_mat1(path, A)


def tsqr_mat1(path, leaf_rows: int = 8192, device=None, chunk_leaves: int | None = None,
              split: bool = True):
    """R (numpy, n x n) of the R-only TSQR of the matrix in a MAT1 file,
    streamed from disk (same leaves and tree as ``tsqr.tsqr`` on the loaded
    matrix, so the same R bit for bit).  NaN/Inf raise ValueError (device flag)."""
    from .core import BlockRowLayout, DimensionError
    from .stream import tsqr_stream
    from .tsqr import MAX_N, _leaves_for, _out, split_leaves

    A = open_mat1(path)
    m, n = A.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if n < 1 or n > MAX_N:
        raise DimensionError(f"GPU TSQR supports 1 <= n <= {MAX_N}, got n = {n}")
    P = _leaves_for(m, n, leaf_rows)
    if split:
        P *= split_leaves(m, n, P, fill=n > 8)
    BlockRowLayout(m, n, P)
    return _out(tsqr_stream(A, P, chunk_leaves=chunk_leaves, device=device), True)
