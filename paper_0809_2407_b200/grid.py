"""CAQR on a Pr x Pc process grid: Algorithm 3.

One rank per GPU; rank (r, c) = r * Pc + c owns the b x b blocks (i, j) with
(i mod Pr, j mod Pc) = (r, c) (``BlockCyclicLayout``, core.py:64-91), stored
as one local row-major matrix (local block (i // Pr, j // Pc)).  For panel j
(block column j, held by process column cj = j mod Pc):

1. TSQR of the panel over the process column (Alg. 3 line 2): each rank
   with active rows (block rows >= j) factors its piece on the GPU (local
   leaves + local tree, implicit Q kept), then the column tree combines the
   R factors with the diagonal-block owner as root (reduce variant, "the
   panel's R factor need only be stored on one processor").
2. Row broadcast (line 3): the factor of each piece -- leaf Y, tau, local
   tree factors and the rank's cross-tree node factors -- goes to the other
   ranks of its process row.
3. Leaf-level update (line 4): every rank applies its row's Q^T to its
   local trailing blocks.
4. Tree-level updates (lines 5-10): per process column, the top b rows of
   the trailing blocks go up the column tree; the receiver applies the node's
   Q^T to [C_a; C_b] and returns the partner's part (``dist.cross_apply``).

Compute is a backend object (``GpuBackend`` drives the sm_100a kernels); the
communication pattern is backend independent, which is what the gloo tests
exercise with an injected CPU backend.  R ends in the upper triangle of the
distributed matrix (diagonal blocks on their owners); ``gather_R`` assembles
it on rank 0.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .core import BlockCyclicLayout, BlockRowLayout, DimensionError
from .dist import broadcast, cross_apply, cross_tree, recv, send
from .trees import BINARY, ReductionTree


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


@dataclass
class GridInfo:
    layout: BlockCyclicLayout
    r: int
    c: int
    row_group: object
    col_group: object

    @property
    def b(self) -> int:
        return self.layout.b

    def local_blocks(self):
        L = self.layout
        return (max(0, _cdiv(L.m_blocks - self.r, L.Pr)), max(0, _cdiv(L.n_blocks - self.c, L.Pc)))

    def first_local_row_block(self, j: int, r: int | None = None) -> int:
        """Local index of the first block row >= j held by process row r."""
        r = self.r if r is None else r
        return max(0, _cdiv(j - r, self.layout.Pr))

    def active_rows(self, j: int, r: int | None = None) -> int:
        r = self.r if r is None else r
        mb = max(0, _cdiv(self.layout.m_blocks - r, self.layout.Pr))
        return max(0, mb - self.first_local_row_block(j, r)) * self.b

    def panel_members(self, j: int):
        """Process rows with active rows for panel j, diagonal owner first."""
        Pr = self.layout.Pr
        rd = j % Pr
        return [(rd + k) % Pr for k in range(Pr) if self.active_rows(j, (rd + k) % Pr) > 0]

    def first_local_col_block(self, jmin: int) -> int:
        """Local index of the first block column >= jmin held by this process column."""
        return max(0, _cdiv(jmin - self.c, self.layout.Pc))


def make_grid(layout: BlockCyclicLayout, backend: str | None = None) -> GridInfo:
    """Row / column communicators of the Pr x Pc grid over the default group."""
    world = dist.get_world_size()
    if world != layout.Pr * layout.Pc:
        raise DimensionError(f"grid {layout.Pr}x{layout.Pc} needs {layout.Pr * layout.Pc} ranks, have {world}")
    rank = dist.get_rank()
    r, c = divmod(rank, layout.Pc)
    row_group = col_group = None
    for rr in range(layout.Pr):  # every rank creates every group, in the same order
        g = dist.new_group([rr * layout.Pc + cc for cc in range(layout.Pc)], backend=backend)
        if rr == r:
            row_group = g
    for cc in range(layout.Pc):
        g = dist.new_group([rr * layout.Pc + cc for rr in range(layout.Pr)], backend=backend)
        if cc == c:
            col_group = g
    return GridInfo(layout, r, c, row_group, col_group)


def scatter_local(A: torch.Tensor, grid: GridInfo) -> torch.Tensor:
    """This rank's local matrix of the block-cyclic distribution of A."""
    L, b = grid.layout, grid.b
    mb, nb = grid.local_blocks()
    out = torch.empty((mb * b, nb * b), dtype=torch.float64, device=A.device)
    for li in range(mb):
        i = grid.r + li * L.Pr
        for lj in range(nb):
            j = grid.c + lj * L.Pc
            out[li * b:(li + 1) * b, lj * b:(lj + 1) * b] = A[i * b:(i + 1) * b, j * b:(j + 1) * b]
    return out


@dataclass
class GridCaqrResult:
    local: torch.Tensor          # this rank's blocks; R in the global upper triangle
    grid: GridInfo
    panels: dict = field(default_factory=dict)   # j -> (local factor, cross nodes) on ranks that hold them
    recorder: object = None
    broadcast_words: int = 0
    R: object = None             # gathered R on rank 0 (set by caqr.caqr_factor)


class GpuBackend:
    """sm_100a kernels for the per-rank compute of grid CAQR."""

    def __init__(self, leaf_rows: int = 2048, device=None, panel_chains: int = 4):
        self.leaf_rows = leaf_rows
        self.device = device
        self.panel_chains = panel_chains

    def _leaves(self, m_r: int, b: int) -> int:
        """caqr_factor's panel leaves: leaf_rows blocks split into up to
        ``panel_chains`` GPU chains (a deeper binary tree of the same TSQR)."""
        from .caqr import _panel_leaves

        P = _panel_leaves(m_r, b, self.leaf_rows)
        while self.panel_chains > 1 and P < self.panel_chains and m_r // (2 * P) >= max(256, 2 * b):
            P *= 2
        return P

    def local_factor(self, piece: torch.Tensor):
        from .tsqr import factor_device

        m_r, b = piece.shape
        # no host-synchronising NaN check per panel (it would stall the
        # lookahead's enqueue order): the flags are checked once at the end
        f = factor_device(piece.contiguous(), self._leaves(m_r, b), want_q=True, check=False)
        self.flags = getattr(self, "flags", [])
        self.flags.append(f.flag)
        return f, f.R.clone()

    def check_finite(self):
        from .tsqr import _check_flag

        for fl in getattr(self, "flags", []):
            _check_flag(fl)
        self.flags = []

    def combine(self, Ra, Rb):
        from .dist import gpu_combine

        return gpu_combine(Ra, Rb)

    def apply_node(self, node, Ca, Cb, transpose):
        from .dist import gpu_apply_node

        return gpu_apply_node(node, Ca, Cb, transpose)

    def local_apply(self, f, C, transpose):
        from .tsqr import apply_q_device

        return apply_q_device(f, C.contiguous(), transpose)

    def local_apply_qt_(self, f, C):
        """Q^T C in place on the strided view of the local trailing blocks."""
        from .tsqr import apply_qt_inplace

        apply_qt_inplace(f, C)

    def pack(self, f, nodes):
        ts = [f.Y, f.tau]
        if f.node_Y is not None:
            ts += [f.node_Y, f.node_tau]
        for (_, _, (Yn, tn)) in nodes:
            ts += [Yn, tn]
        return [t.contiguous() for t in ts]

    def shapes(self, m_r: int, b: int, node_keys):
        from . import _lib
        from .tsqr import _tiles_per_leaf

        P = self._leaves(m_r, b)
        _, h0, ht = _lib.geometry(b)
        tiles = _tiles_per_leaf(BlockRowLayout(m_r, b, P), h0, ht)
        out = [(m_r, b), (P, tiles, b)]
        if P > 1:
            out += [(P - 1, b, b), (P - 1, b)]
        for _ in node_keys:
            out += [(b, b), (b,)]
        return out

    def unpack(self, ts, m_r: int, b: int, node_keys):
        from . import _lib
        from .tsqr import TsqrFactor, _levels_on

        P = self._leaves(m_r, b)
        _, h0, ht = _lib.geometry(b)
        tree = ReductionTree(P=P, shape=BINARY)
        k = 2
        nY = nt = None
        if P > 1:
            nY, nt = ts[2], ts[3]
            k = 4
        f = TsqrFactor(tree=tree, layout=BlockRowLayout(m_r, b, P),
                       R=torch.zeros((b, b), dtype=torch.float64, device=ts[0].device), n=b, h0=h0,
                       ht=ht, Y=ts[0], tau=ts[1], node_Y=nY, node_tau=nt,
                       levels=_levels_on(tree, ts[0].device))
        nodes = []
        for (lvl, partner) in node_keys:
            nodes.append((lvl, partner, (ts[k], ts[k + 1])))
            k += 2
        return f, nodes


def _node_keys(n_members: int, v: int):
    """(level, partner) of the events where virtual index v receives."""
    tree = ReductionTree(P=n_members)
    return [(lvl, b) for lvl, grp in enumerate(tree.levels, start=1) for (a, b) in grp if a == v]


def caqr_grid(local: torch.Tensor, grid: GridInfo, backend, recorder=None,
              lookahead: bool = False) -> GridCaqrResult:
    """Algorithm 3 on this rank's local blocks (modified in place).

    ``lookahead`` (CUDA, opt-in; on a 1 x 1 grid it measured 684 vs 550 ms
    for C5, so it is off by default): Q_j^T is applied to block column j+1 first
    ("near", high-priority stream, with its tree-level exchange), so panel j+1
    is factored while the rest of panel j's trailing update ("far": the
    leaf-level update on a low-priority stream) runs; panel j's far tree-level
    exchange is issued after panel j+1's factor and broadcasts.  Every rank
    issues its collectives in the same order, and the data dependencies are
    the sequential algorithm's, so R is the same as without lookahead.
    """
    L = grid.layout
    b = grid.b
    if L.m < L.n:
        raise DimensionError(f"need m >= n, got {L.m} x {L.n}")
    if L.Pr & (L.Pr - 1):
        raise DimensionError(f"Pr must be a power of two (PAPER.md Alg. 3), got {L.Pr}")
    mb, nb = grid.local_blocks()
    if tuple(local.shape) != (mb * b, nb * b):
        raise DimensionError("local matrix does not match the grid layout")
    res = GridCaqrResult(local=local, grid=grid, recorder=recorder)
    dev = local.device
    if lookahead and dev.type == "cuda":
        _caqr_grid_lookahead(local, grid, backend, recorder, res)
        return res
    for j in range(L.n_blocks):
        cj = j % L.Pc
        members = grid.panel_members(j)
        m_r = grid.active_rows(j)
        mine = m_r > 0
        t0 = grid.first_local_row_block(j) * b
        v = members.index(grid.r) if mine else None
        keys = _node_keys(len(members), v) if mine else []
        f = nodes = None
        # 1. panel TSQR over process column cj
        if grid.c == cj and mine:
            lj = j // L.Pc
            piece = local[t0:, lj * b:(lj + 1) * b]
            f, R = backend.local_factor(piece)
            Rroot, nodes = cross_tree(R, backend.combine, group=grid.col_group, members=members,
                                      recorder=recorder)
            piece.zero_()
            if Rroot is not None:  # diagonal owner: R_jj on the diagonal block
                local[t0:t0 + b, lj * b:(lj + 1) * b] = torch.triu(Rroot)
        # 2. row broadcast of the factors of this process row's piece
        if mine and L.Pc > 1:
            if grid.c == cj:
                ts = backend.pack(f, nodes)
            else:
                ts = [torch.empty(s, dtype=torch.float64, device=dev)
                      for s in backend.shapes(m_r, b, keys)]
            for t in ts:
                broadcast(t, group=grid.row_group, group_src=cj)
                res.broadcast_words += t.numel() if grid.c == cj else 0
            if grid.c != cj:
                f, nodes = backend.unpack(ts, m_r, b, keys)
        if mine:
            res.panels[j] = (f, nodes)
        # 3. leaf-level update of the local trailing blocks (block columns > j)
        lc0 = grid.first_local_col_block(j + 1) * b
        if not mine or lc0 >= local.shape[1]:
            continue
        if hasattr(backend, "local_apply_qt_"):  # in place: no copy of the trailing matrix
            backend.local_apply_qt_(f, local[t0:, lc0:])
        else:
            local[t0:, lc0:] = backend.local_apply(f, local[t0:, lc0:], True)
        # 4. tree-level updates up the column tree (every process column)
        top = cross_apply(nodes, local[t0:t0 + b, lc0:].clone(), backend.apply_node, True,
                          group=grid.col_group, members=members, recorder=recorder)
        local[t0:t0 + b, lc0:] = top
    if hasattr(backend, "check_finite"):
        backend.check_finite()
    return res


def _panel_factor(local, grid, backend, recorder, res, j):
    """Steps 1-2 of Algorithm 3 for panel j: TSQR over process column j mod Pc
    (reduce to the diagonal owner) and the row broadcast of the factors."""
    L, b = grid.layout, grid.b
    cj = j % L.Pc
    members = grid.panel_members(j)
    m_r = grid.active_rows(j)
    mine = m_r > 0
    t0 = grid.first_local_row_block(j) * b
    v = members.index(grid.r) if mine else None
    keys = _node_keys(len(members), v) if mine else []
    f = nodes = None
    if grid.c == cj and mine:
        lj = j // L.Pc
        piece = local[t0:, lj * b:(lj + 1) * b]
        f, R = backend.local_factor(piece)
        Rroot, nodes = cross_tree(R, backend.combine, group=grid.col_group, members=members,
                                  recorder=recorder)
        piece.zero_()
        if Rroot is not None:
            local[t0:t0 + b, lj * b:(lj + 1) * b] = torch.triu(Rroot)
    if mine and L.Pc > 1:
        if grid.c == cj:
            ts = backend.pack(f, nodes)
        else:
            ts = [torch.empty(sh, dtype=torch.float64, device=local.device)
                  for sh in backend.shapes(m_r, b, keys)]
        for t in ts:
            broadcast(t, group=grid.row_group, group_src=cj)
            res.broadcast_words += t.numel() if grid.c == cj else 0
        if grid.c != cj:
            f, nodes = backend.unpack(ts, m_r, b, keys)
    if mine:
        res.panels[j] = (f, nodes)
    return f, nodes, members, mine, t0


def _update(local, grid, backend, recorder, f, nodes, members, t0, lo, hi, tree_level=True):
    """Leaf-level Q^T on local columns [lo, hi) (rows t0:), then the column
    tree's exchange of their top b rows (steps 3-4 of Algorithm 3)."""
    b = grid.b
    if lo < hi:
        C = local[t0:, lo:hi]
        if hasattr(backend, "local_apply_qt_"):
            backend.local_apply_qt_(f, C)
        else:
            local[t0:, lo:hi] = backend.local_apply(f, C, True)
    if tree_level:
        top = cross_apply(nodes, local[t0:t0 + b, lo:hi].clone(), backend.apply_node, True,
                          group=grid.col_group, members=members, recorder=recorder)
        local[t0:t0 + b, lo:hi] = top


def _caqr_grid_lookahead(local, grid, backend, recorder, res):
    """Depth-1 lookahead with the stream structure of caqr.caqr_factor: sA
    (high priority) runs panel j's near update (block column j+1, after panel
    j-1's far update) and factors panel j+1; sB runs panel j's far leaf-level
    update while that happens, then its far tree-level exchange once panel
    j+1's factor (and its communication) is done, so the collectives on each
    communicator execute in the order every rank enqueues them."""
    L, b = grid.layout, grid.b
    width = local.shape[1]
    dev = local.device
    sA = torch.cuda.Stream(device=dev, priority=-1)
    sB = torch.cuda.Stream(device=dev, priority=0)
    cur = torch.cuda.current_stream(dev)
    sA.wait_stream(cur)
    sB.wait_stream(cur)
    nb = L.n_blocks
    fac = [None] * nb
    with torch.cuda.stream(sA):
        fac[0] = _panel_factor(local, grid, backend, recorder, res, 0)
    evB = None
    for j in range(nb):
        f, nodes, members, mine, t0 = fac[j]
        lc0 = grid.first_local_col_block(j + 1) * b if mine else width
        near_hi = lc0 + b if (lc0 < width and (j + 1) % L.Pc == grid.c) else lc0
        with torch.cuda.stream(sA):
            if evB is not None:
                sA.wait_event(evB)
            if mine and near_hi > lc0:
                _update(local, grid, backend, recorder, f, nodes, members, t0, lc0, near_hi)
            evN = torch.cuda.Event()
            evN.record(sA)
        # far leaf-level update enqueued before the next panel's factor (whose
        # communication may block the host), so it overlaps that factor
        with torch.cuda.stream(sB):
            sB.wait_event(evN)
            if mine and near_hi < width:
                _update(local, grid, backend, recorder, f, nodes, members, t0, near_hi, width,
                        tree_level=False)
        with torch.cuda.stream(sA):
            if j + 1 < nb:
                fac[j + 1] = _panel_factor(local, grid, backend, recorder, res, j + 1)
            evF = torch.cuda.Event()
            evF.record(sA)
        with torch.cuda.stream(sB):
            sB.wait_event(evF)
            if mine and near_hi < width:
                top = cross_apply(nodes, local[t0:t0 + b, near_hi:width].clone(), backend.apply_node,
                                  True, group=grid.col_group, members=members, recorder=recorder)
                local[t0:t0 + b, near_hi:width] = top
            evB = torch.cuda.Event()
            evB.record(sB)
    cur.wait_stream(sA)
    cur.wait_stream(sB)
    if hasattr(backend, "check_finite"):
        backend.check_finite()


def gather_R(res: GridCaqrResult):
    """n x n R on rank 0 (None elsewhere), from the blocks (i, j), i <= j < n_blocks."""
    grid = res.grid
    L, b = grid.layout, grid.b
    world = dist.get_world_size()
    rank = dist.get_rank()
    nbk = L.n_blocks

    def rows_of(r):
        return min(max(0, _cdiv(L.m_blocks - r, L.Pr)), max(0, _cdiv(nbk - r, L.Pr))) * b

    def cols_of(c):
        return max(0, _cdiv(nbk - c, L.Pc)) * b

    if rank != 0:
        mine = res.local[:rows_of(grid.r), :cols_of(grid.c)].contiguous()
        if mine.numel():
            send(mine, dst=0)
        return None
    R = torch.zeros((L.n, L.n), dtype=torch.float64, device=res.local.device)
    for src in range(world):
        r, c = divmod(src, L.Pc)
        shape = (rows_of(r), cols_of(c))
        if shape[0] * shape[1] == 0:
            continue
        if src == 0:
            blk = res.local[:shape[0], :shape[1]]
        else:
            blk = torch.empty(shape, dtype=torch.float64, device=res.local.device)
            recv(blk, src=src)
        for li in range(shape[0] // b):
            i = r + li * L.Pr
            for lj in range(shape[1] // b):
                jj = c + lj * L.Pc
                if i <= jj:
                    R[i * b:(i + 1) * b, jj * b:(jj + 1) * b] = blk[li * b:(li + 1) * b,
                                                                    lj * b:(lj + 1) * b]
    return torch.triu(R)
