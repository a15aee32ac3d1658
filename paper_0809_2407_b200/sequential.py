"""Sequential flat-tree TSQR over a block store (Algorithm 2,
PAPER.md:840-866).

``tsqr_sequential(store, layout)`` runs Algorithm 2 literally: load block A_0
and factor it (qr_unblocked), then for every later block load A_k and factor
[R; A_k] (qr_triangle_on_rect, householder.py:297-332), writing each block's
reflectors Y_0k and tau_0k back to the store.  Every factorization runs on the
GPU (the kernel-level API: the shared-memory block kernels up to 128 rows, the
general geqr2 kernel beyond); the store is the "slow memory" of the paper and
its counters record exactly what moves (each A block read once, each Y block
written once).  ``choose_P_sequential`` is the paper's block-count rule
(section 4.2: the smallest P with mn/P + n(n+1)/2 <= W).

The BlockStore is in memory or a directory in the SPEC's on-disk layout
(SPEC.md:333-334): ``meta.json`` (m, n, P, block row counts) and per block
``A_k.mat``, ``Y_k.mat``, ``tau_k.vec`` in MAT1 format (matio.py).

For matrices that live in host memory the binary-tree streamed path
(``stream.tsqr_stream``) is the fast one; this module is the SPEC's
sequential algorithm and its transfer accounting.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

from .core import BlockRowLayout, DimensionError, as_matrix, partition_block_rows


class BlockStore:
    """Blocks A_k, Y_k, tau_k in memory (``directory=None``) or on disk, with
    transfer counters (blocks and words read / written)."""

    def __init__(self, directory: str | None = None):
        self.directory = directory
        self._mem: dict = {}
        self.meta: dict = {}
        self.blocks_read = 0
        self.blocks_written = 0
        self.words_read = 0
        self.words_written = 0
        if directory is not None:
            os.makedirs(directory, exist_ok=True)
            mp = os.path.join(directory, "meta.json")
            if os.path.exists(mp):
                with open(mp) as fh:
                    self.meta = json.load(fh)

    @classmethod
    def from_matrix(cls, A, P: int, directory: str | None = None) -> "BlockStore":
        """Split A into ``BlockRowLayout(m, n, P)`` blocks (core.py:94-102) and
        store them (not counted as transfers: this is the input's creation)."""
        A = as_matrix(A)
        m, n = A.shape
        st = cls(directory)
        blocks = partition_block_rows(A, P)
        st.meta = {"m": m, "n": n, "P": P, "block_rows": [int(b.shape[0]) for b in blocks]}
        for k, b in enumerate(blocks):
            st._put(f"A_{k}", b)
        st._save_meta()
        return st

    # -- raw storage ---------------------------------------------------------
    def _path(self, key):
        ext = ".vec" if key.startswith("tau_") else ".mat"
        return os.path.join(self.directory, key + ext)

    def _put(self, key, arr):
        arr = np.asarray(arr, dtype=np.float64)
        if self.directory is None:
            self._mem[key] = arr.copy()
            return
        from .matio import write_mat1

        write_mat1(self._path(key), arr.reshape(-1, 1) if arr.ndim == 1 else arr)

    def _get(self, key):
        if self.directory is None:
            return self._mem[key].copy()
        from .matio import read_mat1

        arr = read_mat1(self._path(key))
        return arr[:, 0].copy() if key.startswith("tau_") else arr

    def _save_meta(self):
        if self.directory is not None:
            with open(os.path.join(self.directory, "meta.json"), "w") as fh:
                json.dump(self.meta, fh)

    # -- counted transfers -----------------------------------------------------
    @property
    def P(self) -> int:
        return int(self.meta["P"])

    def read_block(self, k: int) -> np.ndarray:
        a = self._get(f"A_{k}")
        self.blocks_read += 1
        self.words_read += a.size
        return a

    def write_factor(self, k: int, Y: np.ndarray, tau: np.ndarray) -> None:
        self._put(f"Y_{k}", Y)
        self._put(f"tau_{k}", tau)
        self.blocks_written += 1
        self.words_written += int(np.asarray(Y).size + np.asarray(tau).size)

    def read_factor(self, k: int):
        return self._get(f"Y_{k}"), self._get(f"tau_{k}")

    def counters(self) -> dict:
        return {"blocks_read": self.blocks_read, "blocks_written": self.blocks_written,
                "words_read": self.words_read, "words_written": self.words_written}


def choose_P_sequential(m: int, n: int, W: int) -> int:
    """Smallest P with mn/P + n(n+1)/2 <= W (section 4.2)."""
    tri = n * (n + 1) // 2
    if W <= tri:
        raise ValueError("matrix column count too large for fast memory")
    return max(1, -(-(m * n) // (W - tri)))


@dataclass
class SequentialTsqrFactor:
    """TsqrFactor of the flat tree: the chain factors
    Y_0k / tau_0k live in the store; R is the final triangle."""

    R: np.ndarray
    layout: BlockRowLayout
    store: BlockStore = field(repr=False)
    host: bool = True

    @property
    def n(self) -> int:
        return self.R.shape[0]

    @property
    def m(self) -> int:
        return self.layout.m

    def _factor(self, k):
        from .householder import DENSE, TRI_ON_RECT, HouseholderFactor

        Y, tau = self.store.read_factor(k)
        if k == 0:
            return HouseholderFactor(Y, tau, DENSE)
        return HouseholderFactor(Y, tau, TRI_ON_RECT, rows_rect=Y.shape[0])

    def apply_q(self, C, transpose: bool = False):
        """Q C / Q^T C with Q = Q_00 Q_01 ... Q_0,P-1 (each Q_0k acting on the n
        pivot rows and block k's rows; apply_q / apply_qt of each factor)."""
        from .householder import apply_q

        C = np.array(as_matrix(C, "C"), copy=True)
        offs = self.layout.row_offsets()
        n = self.n
        if C.shape[0] != self.m:
            raise DimensionError(f"C has {C.shape[0]} rows, factor acts on {self.m}")
        order = range(self.layout.P) if transpose else reversed(range(self.layout.P))
        for k in order:
            f = self._factor(k)
            if k == 0:
                C[offs[0]:offs[1]] = apply_q(f, C[offs[0]:offs[1]], transpose)
            else:
                rows = np.concatenate([np.arange(n), np.arange(offs[k], offs[k + 1])])
                C[rows] = apply_q(f, C[rows], transpose)
        return C

    def explicit_q(self):
        E = np.zeros((self.m, self.n))
        E[:self.n, :self.n] = np.eye(self.n)
        return self.apply_q(E)


def tsqr_sequential(store: BlockStore, layout: BlockRowLayout | None = None,
                    counter=None) -> SequentialTsqrFactor:
    """Algorithm 2 over the store's blocks: R in fast memory,
    the Y / tau chain written back block by block."""
    from .householder import qr_triangle_on_rect, qr_unblocked

    meta = store.meta
    m, n, P = int(meta["m"]), int(meta["n"]), int(meta["P"])
    lay = layout if layout is not None else BlockRowLayout(m, n, P)
    if (lay.m, lay.n, lay.P) != (m, n, P):
        raise DimensionError("layout does not match the store")
    A0 = store.read_block(0)
    if A0.shape[0] < n:
        raise DimensionError(f"block 0 has {A0.shape[0]} rows, fewer than n = {n}")
    f0, R = qr_unblocked(A0, counter)
    store.write_factor(0, f0.Y, f0.tau)
    for k in range(1, P):
        Ak = store.read_block(k)
        fk, R = qr_triangle_on_rect(R, Ak, counter)
        store.write_factor(k, fk.Y, fk.tau)
    return SequentialTsqrFactor(np.asarray(R), lay, store)
