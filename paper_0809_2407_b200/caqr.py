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
    launches: int = 0            # kernels of this library launched by the factorization

    @property
    def R(self):
        return _out(torch.triu(self.W[: self.n, : self.n]), self.host)


def _panel_leaves(mj: int, w: int, leaf_rows: int) -> int:
    P = max(1, mj // max(1, leaf_rows))
    while P > 1 and mj // P < w:
        P -= 1
    return P


def caqr_factor(A, layout: BlockCyclicLayout | None = None, b: int = 128, leaf_rows: int = 2048,
                device=None, counter=None, lookahead: bool = True,
                panel_chains: int = 4, apply_waves: float = 4.0) -> CaqrResult:
    """CAQR of A (m x n, m >= n) with panel width b <= 128.

    With ``lookahead`` (default) the panels run on a high-priority stream:
    panel j+1's columns are updated by Q_j and factored there while the
    low-priority stream applies Q_j to the rest of the trailing matrix
    (depth-1 lookahead; the data dependencies are the same as the
    sequential right-looking order, so results are identical).  The panel
    factor then only needs a few SMs' worth of work to hide behind the
    trailing update; ``panel_chains`` splits each panel leaf into that many
    ring chains (a deeper binary tree, see tsqr.split_leaves).

    ``apply_waves``: the trailing update runs one CTA per (panel leaf, 128
    trailing columns); as the trailing matrix shrinks, a panel's leaves are
    split (more, shorter leaves: the same binary-tree TSQR with more events)
    until its update fills that many waves of the SMs, so the late panels do
    not run on a handful of SMs.  0 keeps ``leaf_rows`` leaves throughout.
    """
    lib = _lib.load()
    if layout is not None:
        b = layout.b
        if layout.Pr * layout.Pc > 1:
            return _caqr_on_grid(A, layout, leaf_rows, device)
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
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    starts = list(range(0, n, b))
    nb = len(starts)
    panels = [None] * nb
    nlaunch = [0]
    # plan every panel and carve all device buffers out of four allocations up
    # front, so the enqueue loop below never allocates (no allocator stalls
    # between the two streams)
    plan = []
    n_tau = n_rs = n_ny = n_nt = 0
    for c0 in starts:
        c1 = min(c0 + b, n)
        w = c1 - c0
        mj = m - c0
        P = _panel_leaves(mj, w, leaf_rows)
        while panel_chains > 1 and P < panel_chains and mj // (2 * P) >= max(256, 2 * w):
            P *= 2  # split leaves into GPU chains (hybrid tree, see tsqr.split_leaves)
        if apply_waves > 0 and c1 < n:
            want = apply_waves * sms / max(1, -(-(n - c1) // 128))
            while P < want and mj // (2 * P) >= max(256, 2 * w):
                P *= 2
        lay = BlockRowLayout(mj, w, P)
        _, h0, ht = _lib.geometry(w)
        tiles = _tiles_per_leaf(lay, h0, ht)
        tree = ReductionTree(P=P, shape=BINARY)
        plan.append((c0, c1, w, mj, P, lay, h0, tiles, tree, _levels_on(tree, dev),
                     n_tau, n_rs, n_ny, n_nt))
        n_tau += P * tiles * w
        n_rs += P * w * w
        n_ny += (P - 1) * w * w
        n_nt += (P - 1) * w
    # panel T of the chain tiles (tsqr_f64_leaf_factor_t / _apply_t): two slots, panel jp uses
    # slot jp & 1 -- factor(jp + 1) is enqueued behind the far update of panel jp - 1 (evB), the
    # last reader of that slot
    use_t = bool(lib.tsqr_f64_panel_t_used(b)) if nb > 1 else False
    t_len = max((pl[4] * pl[7] for pl in plan), default=0) * 1024 if use_t else 0
    t_all = torch.empty((2, max(1, t_len)), dtype=torch.float64, device=dev)
    tau_all = torch.zeros(max(1, n_tau), dtype=torch.float64, device=dev)
    rs_all = torch.empty(max(1, n_rs), dtype=torch.float64, device=dev)
    ny_all = torch.zeros(max(1, n_ny), dtype=torch.float64, device=dev)
    nt_all = torch.zeros(max(1, n_nt), dtype=torch.float64, device=dev)
    roots = [None] * nb

    def factor(jp, st):
        c0, c1, w, mj, P, lay, h0, tiles, tree, levels, o_t, o_r, o_y, o_n = plan[jp]
        tau = tau_all[o_t:o_t + P * tiles * w].view(P, tiles, w)
        Rs = rs_all[o_r:o_r + P * w * w].view(P, w, w)
        base_ptr = _ptr(W) + 8 * (c0 * n + c0)
        sh = int(st.cuda_stream)
        nlaunch[0] += 1 + (mj - lay.base * (P - 1) > h0) + (len(levels) if P > 1 else 0)
        if use_t and w == b:
            _lib.check(lib.tsqr_f64_leaf_factor_t(base_ptr, n, mj, w, P, base_ptr, n, _ptr(tau),
                                                  tiles * w, _ptr(Rs), _ptr(flag),
                                                  _ptr(t_all[jp & 1]), sh),
                       "tsqr_f64_leaf_factor_t")
        else:
            _lib.check(lib.tsqr_f64_leaf_factor(base_ptr, n, mj, w, P, base_ptr, n, _ptr(tau),
                                                tiles * w, _ptr(Rs), _ptr(flag), sh),
                       "tsqr_f64_leaf_factor")
        node_Y = node_tau = None
        if P > 1:
            node_Y = ny_all[o_y:o_y + (P - 1) * w * w].view(P - 1, w, w)
            node_tau = nt_all[o_n:o_n + (P - 1) * w].view(P - 1, w)
            for ev in levels:
                _lib.check(lib.tsqr_f64_tree_factor_level(_ptr(Rs), w, _ptr(ev), ev.shape[0],
                                                          _ptr(node_Y), _ptr(node_tau), sh),
                           "tsqr_f64_tree_factor_level")
        # the root R goes onto the diagonal block after the loop (no later
        # panel reads it); its strict lower part keeps leaf 0's Y
        roots[jp] = Rs[tree.root]
        panels[jp] = CaqrPanel(c0, c1, lay, tree, tau, node_Y, node_tau, levels)

    def apply(jp, lo, hi, st):
        """Q_jp^T applied to W[c0:, lo:hi] (leaf level, then the tree levels)."""
        if lo >= hi:
            return
        pnl = panels[jp]
        c0, w, P = pnl.c0, pnl.width, pnl.layout.P
        mj = m - c0
        base_ptr = _ptr(W) + 8 * (c0 * n + c0)
        cptr = _ptr(W) + 8 * (c0 * n + lo)
        sh = int(st.cuda_stream)
        nlaunch[0] += 1 + len(pnl.levels)
        if use_t and w == b:
            _lib.check(lib.tsqr_f64_leaf_apply_t(base_ptr, n, _ptr(pnl.tau), pnl.tau.shape[1] * w,
                                                 mj, w, P, cptr, n, hi - lo, _ptr(t_all[jp & 1]),
                                                 sh),
                       "tsqr_f64_leaf_apply_t")
        else:
            _lib.check(lib.tsqr_f64_leaf_apply(base_ptr, n, _ptr(pnl.tau), pnl.tau.shape[1] * w, mj,
                                               w, P, cptr, n, hi - lo, 0, 0, 0, 1, 0, 0, sh),
                       "tsqr_f64_leaf_apply")
        for ev in pnl.levels:
            _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(pnl.node_Y), _ptr(pnl.node_tau), w,
                                                     _ptr(ev), ev.shape[0], cptr, n,
                                                     pnl.layout.base, hi - lo, 1, 0, sh),
                       "tsqr_f64_tree_apply_level")

    cur = torch.cuda.current_stream(dev)
    if not lookahead or nb == 1:
        for jp in range(nb):
            factor(jp, cur)
            if jp + 1 < nb:
                apply(jp, starts[jp + 1], n, cur)
    else:
        sA = torch.cuda.Stream(device=dev, priority=-1)
        sB = torch.cuda.Stream(device=dev, priority=0)
        sA.wait_stream(cur)
        sB.wait_stream(cur)
        evF = [None] * nb
        evB = [None] * nb
        factor(0, sA)
        evF[0] = torch.cuda.Event()
        evF[0].record(sA)
        for jp in range(nb):
            if jp + 1 < nb:
                # near: block jp+1 already carries Q_0..Q_{jp-1} (far updates on sB)
                if jp >= 1:
                    sA.wait_event(evB[jp - 1])
                nxt = starts[jp + 1]
                apply(jp, nxt, min(nxt + b, n), sA)
                factor(jp + 1, sA)
                evF[jp + 1] = torch.cuda.Event()
                evF[jp + 1].record(sA)
            sB.wait_event(evF[jp])
            if jp + 2 < nb:
                apply(jp, starts[jp + 2], n, sB)
            evB[jp] = torch.cuda.Event()
            evB[jp].record(sB)
        cur.wait_stream(sA)
        cur.wait_stream(sB)
    for jp in range(nb):
        c0, c1 = plan[jp][0], plan[jp][1]
        blk = W[c0:c1, c0:c1]
        blk.copy_(torch.tril(blk, -1) + roots[jp])
    _check_flag(flag)
    if counter is not None:
        counter.add(2 * m * n * n - (2 * n ** 3) // 3)
    return CaqrResult(W=W, panels=panels, m=m, n=n, b=b, host=host, launches=nlaunch[0])


_GRIDS: dict = {}


def _caqr_on_grid(A, layout: BlockCyclicLayout, leaf_rows: int, device):
    """Algorithm 3 on the Pr x Pc process grid of the initialised
    torch.distributed job (one rank per GPU, world = Pr * Pc); every rank
    passes the same global A and keeps its own blocks (grid.py)."""
    import torch.distributed as dist

    from .executor import ExecutorError
    from .grid import GpuBackend, caqr_grid, gather_R as grid_gather_R, make_grid, scatter_local

    if not dist.is_initialized() or dist.get_world_size() != layout.Pr * layout.Pc:
        raise ExecutorError(f"a {layout.Pr}x{layout.Pc} layout needs torch.distributed initialised "
                            f"with {layout.Pr * layout.Pc} ranks (one per GPU)")
    At, host = to_device(A, device)
    if (layout.m, layout.n) != tuple(At.shape):
        raise DimensionError("layout does not match A")
    # the grid's row / column groups belong to the default group they were made
    # in: after destroy / re-init the cached groups are dead, so the cache entry
    # keeps that group and is rebuilt when it is no longer the current one
    key = (layout.m, layout.n, layout.b, layout.Pr, layout.Pc)
    world = dist.group.WORLD
    grid, made_in = _GRIDS.get(key, (None, None))
    if grid is None or made_in is not world:  # every rank reaches this in the same order
        grid = make_grid(layout)
        _GRIDS[key] = (grid, world)
    res = caqr_grid(scatter_local(At, grid), grid, GpuBackend(leaf_rows=leaf_rows))
    R = grid_gather_R(res)
    res.R = None if R is None else _out(R, host)
    return res


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
