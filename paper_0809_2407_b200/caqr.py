"""CAQR on B200: right-looking CAQR (Algorithm 3) with
TSQR panels, over the sm_100a kernels.

Per panel j of width b:
  1. TSQR of the panel's active rows: leaves of ``leaf_rows`` rows
     (BlockRowLayout), leaf implicit Q written IN PLACE over the panel
     (LAPACK style), binary tree of stacked-triangle
     combines whose root R lands on the diagonal block (reduce variant).
  2. Leaf-level update of the trailing columns, C <- Q_leaf^T C
     (Alg. 3 line 4; the compact-WY ``_apply_yt(transpose=True)`` of the
     reference, householder.py:175-186, executed reflector-by-reflector on
     chip by the leaf-apply kernel).
  3. Tree-level updates on the leaf top blocks, [C0; C1] <- Q_node^T [C0; C1]
     (Alg. 3 lines 5-10; ``apply_qt_structured``, householder.py:335-374).
The Pr = Pc = 1 case is the SPEC's "degenerates to sequential blocked QR"
(SPEC.md:363); ``layout`` is accepted for API compatibility, the 2-D grid
execution across GPUs is described in DESIGN.md.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import BlockCyclicLayout, BlockRowLayout, DimensionError
from .tsqr import _ptr, _stream, _out, to_device, _tiles_per_leaf, _levels_on, _check_flag
from .trees import BINARY, ReductionTree


@dataclass
class CaqrPanel:
    c0: int
    c1: int
    layout: BlockRowLayout      # leaves over the panel's active rows (rows c0..m)
    tree: ReductionTree
    tau: torch.Tensor            # P x tiles x w
    node_Y: torch.Tensor | None
    node_tau: torch.Tensor | None
    levels: list = field(default_factory=list)

    @property
    def width(self) -> int:
        return self.c1 - self.c0


@dataclass
class CaqrResult:
    """SPEC CaqrResult: R, per-panel TSQR factors, recorders.

    ``W`` (m x n, device) holds R in its upper triangle and every panel's
    leaf implicit Q below it; ``panels`` hold tau and the interior factors.
    """

    W: torch.Tensor
    panels: list
    m: int
    n: int
    b: int
    host: bool = False
    recorders: list = field(default_factory=list)

    @property
    def R(self):
        return _out(torch.triu(self.W[: self.n, : self.n]), self.host)


def _panel_leaves(mj: int, w: int, leaf_rows: int) -> int:
    P = max(1, mj // max(1, leaf_rows))
    while P > 1 and mj // P < w:
        P -= 1
    return P


def caqr_factor(A, layout: BlockCyclicLayout | None = None, b: int = 128, leaf_rows: int = 2048,
                device=None, counter=None) -> CaqrResult:
    """CAQR of A (m x n, m >= n) with panel width b <= 128."""
    lib = _lib.load()
    if layout is not None:
        b = layout.b
    At, host = to_device(A, device)
    m, n = At.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if not 1 <= b <= 128:
        raise DimensionError(f"panel width b must be in [1, 128], got {b}")
    if layout is not None and (layout.m, layout.n) != (m, n):
        raise DimensionError("layout does not match A")
    W = At.clone() if not host else At
    dev = W.device
    st = _stream(dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    panels = []
    for c0 in range(0, n, b):
        c1 = min(c0 + b, n)
        w = c1 - c0
        mj = m - c0
        P = _panel_leaves(mj, w, leaf_rows)
        lay = BlockRowLayout(mj, w, P)
        _, h0, ht = _lib.geometry(w)
        tau = torch.zeros((P, _tiles_per_leaf(lay, h0, ht), w), dtype=torch.float64, device=dev)
        Rs = torch.empty((P, w, w), dtype=torch.float64, device=dev)
        base_ptr = _ptr(W) + 8 * (c0 * n + c0)
        _lib.check(lib.tsqr_f64_leaf_factor(base_ptr, n, mj, w, P, base_ptr, n, _ptr(tau),
                                            tau.shape[1] * w, _ptr(Rs), _ptr(flag), st),
                   "tsqr_f64_leaf_factor")
        tree = ReductionTree(P=P, shape=BINARY)
        levels = _levels_on(tree, dev)
        node_Y = node_tau = None
        if P > 1:
            node_Y = torch.zeros((P - 1, w, w), dtype=torch.float64, device=dev)
            node_tau = torch.zeros((P - 1, w), dtype=torch.float64, device=dev)
            for ev in levels:
                _lib.check(lib.tsqr_f64_tree_factor_level(_ptr(Rs), w, _ptr(ev), ev.shape[0],
                                                          _ptr(node_Y), _ptr(node_tau), st),
                           "tsqr_f64_tree_factor_level")
        # root R onto the diagonal block (its strict lower part keeps leaf 0's Y)
        blk = W[c0:c1, c0:c1]
        blk.copy_(torch.tril(blk, -1) + Rs[tree.root])
        if c1 < n:
            cptr = _ptr(W) + 8 * (c0 * n + c1)
            _lib.check(lib.tsqr_f64_leaf_apply(base_ptr, n, _ptr(tau), tau.shape[1] * w, mj, w, P,
                                               cptr, n, n - c1, 0, 0, 0, 1, 0, 0, st),
                       "tsqr_f64_leaf_apply")
            for ev in levels:
                _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(node_Y), _ptr(node_tau), w, _ptr(ev),
                                                         ev.shape[0], cptr, n, lay.base, n - c1,
                                                         1, 0, st),
                           "tsqr_f64_tree_apply_level")
        panels.append(CaqrPanel(c0, c1, lay, tree, tau, node_Y, node_tau, levels))
    _check_flag(flag)
    if counter is not None:
        counter.add(2 * m * n * n - (2 * n ** 3) // 3)
    return CaqrResult(W=W, panels=panels, m=m, n=n, b=b, host=host)


def gather_R(result: CaqrResult):
    """n x n upper-triangular R."""
    return result.R


def caqr_apply_q(result: CaqrResult, C, transpose: bool = False):
    """Q C or Q^T C (C has m rows) with Q = Q_0 Q_1 ... Q_{panels-1}."""
    lib = _lib.load()
    Ct, host = to_device(C, result.W.device, name="C")
    if Ct.shape[0] != result.m:
        raise DimensionError(f"C has {Ct.shape[0]} rows, factor acts on {result.m}")
    out = Ct.clone()
    k = out.shape[1]
    st = _stream(out.device)
    n = result.n
    order = result.panels if transpose else list(reversed(result.panels))
    for p in order:
        w, mj, P = p.width, result.m - p.c0, p.layout.P
        yptr = _ptr(result.W) + 8 * (p.c0 * n + p.c0)
        cptr = _ptr(out) + 8 * (p.c0 * k)
        if transpose:
            _lib.check(lib.tsqr_f64_leaf_apply(yptr, n, _ptr(p.tau), p.tau.shape[1] * w, mj, w, P,
                                               cptr, k, k, 0, 0, 0, 1, 0, 0, st), "leaf_apply")
            for ev in p.levels:
                _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(p.node_Y), _ptr(p.node_tau), w,
                                                         _ptr(ev), ev.shape[0], cptr, k,
                                                         p.layout.base, k, 1, 0, st), "tree_apply")
        else:
            for ev in reversed(p.levels):
                _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(p.node_Y), _ptr(p.node_tau), w,
                                                         _ptr(ev), ev.shape[0], cptr, k,
                                                         p.layout.base, k, 0, 0, st), "tree_apply")
            _lib.check(lib.tsqr_f64_leaf_apply(yptr, n, _ptr(p.tau), p.tau.shape[1] * w, mj, w, P,
                                               cptr, k, k, 0, 0, 0, 0, 0, 0, st), "leaf_apply")
    return _out(out, host or result.host)
