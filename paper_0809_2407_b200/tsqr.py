"""TSQR on B200: the SPEC's tsqr entry points over the sm_100a kernels.

Follows SPEC.md:259-340 (tsqr module) and Algorithm 1 of the paper
(reduce variant): every leaf row block is factored by one
CTA of ``tsqr_f64_leaf_factor`` (dense first tile + flat chain of
triangle-on-rectangle tiles, Alg. 2 inside the leaf), then the leaf R factors
are combined pairwise up the reduction tree (``tsqr_f64_tree_factor_level``,
one launch per level, events of a level in parallel).  Q stays implicit
(leaf Y / tau, interior STACKED factors) and is applied by walking the tree
back down.

Inputs may be numpy arrays (copied to the GPU; results come back as numpy,
like the reference) or CUDA torch tensors (everything stays on device).
There is no CPU fallback: the CUDA library must load.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import BlockRowLayout, DimensionError
from .counters import count_stacked, count_tri_rect, count_geqr2
from .executor import DeviceExecutor
from .trees import BINARY, ReductionTree, TreeError

MAX_N = 128


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(device) -> int:
    return int(torch.cuda.current_stream(device).cuda_stream)


def to_device(A, device=None, name="matrix"):
    """(float64 contiguous CUDA tensor, was_host) with the reference's checks."""
    if isinstance(A, torch.Tensor):
        if A.ndim != 2:
            raise DimensionError(f"{name} must be 2-D, got ndim={A.ndim}")
        dev = device if device is not None else (A.device if A.is_cuda else torch.device("cuda"))
        t = A.to(device=dev, dtype=torch.float64)
        return t.contiguous(), not A.is_cuda
    arr = np.asarray(A, dtype=np.float64)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got ndim={arr.ndim}")
    dev = device if device is not None else torch.device("cuda")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev), True


def _out(t, host: bool):
    """Result in the caller's memory space: numpy for host callers.  Large
    results go through a pinned buffer (full-bandwidth D2H; the caching host
    allocator recycles it once the array is dropped)."""
    if not host:
        return t
    if t.numel() * t.element_size() < (1 << 22):
        return t.cpu().numpy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()


def _check_flag(flag) -> None:
    if int(flag.item()) != 0:
        raise ValueError("matrix contains NaN or Inf entries")


@dataclass
class TsqrFactor:
    """SPEC TsqrFactor: tree, leaf factors, interior factors,
    final R and layout.  Device tensors:

    * ``Y`` (m x n): leaf implicit Q.  Leaf i's rows hold its dense first tile
      (LAPACK layout: R above / Y strictly below the unit diagonal) followed by
      the rectangles V of its chain tiles (``ht`` rows each).
    * ``tau`` (P x tiles x n): tile t of leaf i at ``tau[i, t]``.
    * ``node_Y`` (P-1 x n x n), ``node_tau`` (P-1 x n): the STACKED factor of
      every combine event in ``tree.schedule()`` order (Y = [I; node_Y]).
    """

    tree: ReductionTree
    layout: BlockRowLayout
    R: torch.Tensor
    n: int
    h0: int
    ht: int
    Y: torch.Tensor | None = None
    tau: torch.Tensor | None = None
    node_Y: torch.Tensor | None = None
    node_tau: torch.Tensor | None = None
    host: bool = False
    levels: list = field(default_factory=list)
    flag: torch.Tensor | None = None

    @property
    def m(self) -> int:
        return self.layout.m

    def check_finite(self) -> None:
        """Raise ValueError if the factored matrix held NaN/Inf (core.py:26-27)."""
        if self.flag is not None:
            _check_flag(self.flag)

    @property
    def P(self) -> int:
        return self.layout.P

    @property
    def has_q(self) -> bool:
        return self.Y is not None

    def R_out(self):
        return _out(self.R, self.host)

    # reference-style views of the implicit Q (host copies, for inspection)
    def interior_factors(self):
        from .householder import HouseholderFactor, STACKED

        out = []
        if self.node_Y is None:
            return out
        Yn, tn = self.node_Y.cpu().numpy(), self.node_tau.cpu().numpy()
        for e in range(Yn.shape[0]):
            Yf = np.vstack([np.eye(self.n), Yn[e]])
            out.append(HouseholderFactor(Yf, tn[e].copy(), shape_tag=STACKED, q=2))
        return out


def _tiles_per_leaf(layout: BlockRowLayout, h0: int, ht: int) -> int:
    b = max(layout.block_rows)
    return 1 + max(0, -(-(b - h0) // ht))


_LEVEL_CACHE: dict = {}


def _levels_on(tree: ReductionTree, device):
    """Per-level event arrays on the device, packed once per (tree, device)."""
    key = (tree.P, tree.shape, tree.levels, str(device))
    lv = _LEVEL_CACHE.get(key)
    if lv is None:
        packed = tree.device_levels()
        if packed:
            flat = torch.from_numpy(np.concatenate(packed)).to(device)
            lv, o = [], 0
            for a in packed:
                lv.append(flat[o:o + len(a)])
                o += len(a)
        else:
            lv = []
        _LEVEL_CACHE[key] = lv
    return lv


def _count(counter, layout, n, h0, ht, P):
    for b in layout.block_rows:
        f, d = count_geqr2(min(b, h0), n)
        counter.add(f, d)
        rest = b - min(b, h0)
        while rest > 0:
            f, d = count_tri_rect(n, min(ht, rest))
            counter.add(f, d)
            rest -= ht
    f, d = count_stacked(n)
    counter.add(f * (P - 1), d * (P - 1))


def factor_device(A: torch.Tensor, P: int, want_q: bool = False, tree: ReductionTree | None = None,
                  Y_out: torch.Tensor | None = None, counter=None, host=False,
                  check: bool = True) -> TsqrFactor:
    """TSQR of a CUDA float64 matrix (m x n, n <= 128) over P leaves.

    ``check=False`` skips the (host-synchronising) NaN/Inf check; the device
    flag is returned as ``factor.flag`` for a deferred ``check_finite`` --
    this is what makes the call capturable in a CUDA graph.
    """
    lib = _lib.load()
    if A.ndim != 2:
        raise DimensionError("A must be 2-D")
    m, n = A.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if n < 1 or n > MAX_N:
        raise DimensionError(f"GPU TSQR supports 1 <= n <= {MAX_N}, got n = {n}")
    layout = BlockRowLayout(m, n, P)
    tree = tree if tree is not None else ReductionTree(P=P, shape=BINARY)
    if tree.P != P:
        raise TreeError(f"tree has {tree.P} leaves, layout has {P}")
    if not A.is_contiguous():
        A = A.contiguous()
    dev = A.device
    _, h0, ht = _lib.geometry(n)
    st = _stream(dev)
    Rs = torch.empty((P, n, n), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if not want_q and tree.shape == BINARY:
        # R only on the binary tree: one C-ABI call, no node factors stored
        nlev = max(1, (P - 1).bit_length())
        tickets = torch.empty(nlev * P, dtype=torch.int32, device=dev)
        _lib.check(lib.tsqr_f64_r_binary(_ptr(A), n, m, n, P, _ptr(Rs), _ptr(tickets), _ptr(flag),
                                         st), "tsqr_f64_r_binary")
        if check:
            _check_flag(flag)
        if counter is not None:
            _count(counter, layout, n, h0, ht, P)
        return TsqrFactor(tree=tree, layout=layout, R=Rs[0], n=n, h0=h0, ht=ht, host=host,
                          flag=flag)
    Y = tau = None
    if want_q:
        Y = Y_out if Y_out is not None else torch.empty_like(A)
        tau = torch.zeros((P, _tiles_per_leaf(layout, h0, ht), n), dtype=torch.float64, device=dev)
    _lib.check(lib.tsqr_f64_leaf_factor(_ptr(A), n, m, n, P, _ptr(Y), n, _ptr(tau),
                                        0 if tau is None else tau.shape[1] * n, _ptr(Rs),
                                        _ptr(flag), st), "tsqr_f64_leaf_factor")
    levels = _levels_on(tree, dev)
    node_Y = node_tau = None
    if P > 1:
        node_Y = torch.zeros((P - 1, n, n), dtype=torch.float64, device=dev)
        node_tau = torch.zeros((P - 1, n), dtype=torch.float64, device=dev)
        for ev in levels:
            _lib.check(lib.tsqr_f64_tree_factor_level(_ptr(Rs), n, _ptr(ev), ev.shape[0],
                                                      _ptr(node_Y), _ptr(node_tau), st),
                       "tsqr_f64_tree_factor_level")
    if check:
        _check_flag(flag)
    if counter is not None:
        _count(counter, layout, n, h0, ht, P)
    return TsqrFactor(tree=tree, layout=layout, R=Rs[tree.root], n=n, h0=h0, ht=ht, Y=Y, tau=tau,
                      node_Y=node_Y, node_tau=node_tau, host=host, levels=levels, flag=flag)


def _tree_apply(f: TsqrFactor, C: torch.Tensor, slot_rows: int, transpose: bool, zero_partner: bool):
    lib = _lib.load()
    if f.P == 1:
        return
    st = _stream(C.device)
    order = f.levels if transpose else list(reversed(f.levels))
    ldc = C.stride(0) if C.dim() == 2 and C.stride(1) == 1 else C.shape[1]
    for ev in order:
        _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(f.node_Y), _ptr(f.node_tau), f.n, _ptr(ev),
                                                 ev.shape[0], _ptr(C), ldc, slot_rows,
                                                 C.shape[1], int(transpose), int(zero_partner), st),
                   "tsqr_f64_tree_apply_level")


def _leaf_apply(f: TsqrFactor, C: torch.Tensor, transpose: bool, S=None, zero_init=False,
                tri_skip=False):
    lib = _lib.load()
    st = _stream(C.device)
    k = C.shape[1]
    ldc = C.stride(0) if C.stride(1) == 1 else k  # strided column slices apply in place
    _lib.check(lib.tsqr_f64_leaf_apply(_ptr(f.Y), f.n, _ptr(f.tau), f.tau.shape[1] * f.n, f.m,
                                       f.n, f.P, _ptr(C), ldc, k, _ptr(S), k,
                                       f.n if S is not None else 0, int(transpose),
                                       int(zero_init), int(tri_skip), st),
               "tsqr_f64_leaf_apply")


def explicit_q_device(f: TsqrFactor) -> torch.Tensor:
    """Thin Q (m x n): Q [I; 0] by walking the tree down, then every leaf chain."""
    if not f.has_q:
        raise ValueError("factor was computed without implicit Q (want_q=False)")
    n, dev = f.n, f.R.device
    S = torch.zeros((f.P, n, n), dtype=torch.float64, device=dev)
    S[f.tree.root] = torch.eye(n, dtype=torch.float64, device=dev)
    _tree_apply(f, S.view(f.P * n, n), slot_rows=n, transpose=False, zero_partner=True)
    Q = torch.empty((f.m, n), dtype=torch.float64, device=dev)
    _leaf_apply(f, Q, transpose=False, S=S.view(f.P * n, n), zero_init=True, tri_skip=True)
    return Q


def apply_qt_inplace(f: TsqrFactor, C: torch.Tensor) -> None:
    """C := Q^T C in place; C (m x k) may be a column slice of a row-major
    matrix (unit column stride, any row stride): no copy of the trailing
    matrix (the CAQR grid's leaf-level update)."""
    if not f.has_q:
        raise ValueError("factor was computed without implicit Q (want_q=False)")
    if C.shape[0] != f.m or C.stride(1) != 1:
        raise DimensionError("C must have the factor's rows and unit column stride")
    _leaf_apply(f, C, transpose=True)
    _tree_apply(f, C, slot_rows=f.layout.base, transpose=True, zero_partner=False)


def apply_q_device(f: TsqrFactor, C: torch.Tensor, transpose: bool) -> torch.Tensor:
    """Q C / Q^T C with the full m x m Q assembled per tree.

    transpose=False: C is n x k (thin: Q_thin C, m x k) or m x k (full).
    transpose=True : C is m x k, returns Q^T C (m x k); its first n rows are
    Q_thin^T C (the root leaf starts at row 0).
    """
    if not f.has_q:
        raise ValueError("factor was computed without implicit Q (want_q=False)")
    n, dev = f.n, f.R.device
    k = C.shape[1]
    if transpose:
        if C.shape[0] != f.m:
            raise DimensionError(f"C has {C.shape[0]} rows, factor acts on {f.m}")
        out = C.clone()
        _leaf_apply(f, out, transpose=True)
        _tree_apply(f, out, slot_rows=f.layout.base, transpose=True, zero_partner=False)
        return out
    if C.shape[0] == n and f.m != n:
        S = torch.zeros((f.P, n, k), dtype=torch.float64, device=dev)
        S[f.tree.root] = C
        _tree_apply(f, S.view(f.P * n, k), slot_rows=n, transpose=False, zero_partner=True)
        out = torch.empty((f.m, k), dtype=torch.float64, device=dev)
        _leaf_apply(f, out, transpose=False, S=S.view(f.P * n, k), zero_init=True)
        return out
    if C.shape[0] != f.m:
        raise DimensionError(f"C has {C.shape[0]} rows; expected {n} (thin) or {f.m} (full)")
    out = C.clone()
    _tree_apply(f, out, slot_rows=f.layout.base, transpose=False, zero_partner=False)
    _leaf_apply(f, out, transpose=False)
    return out


# ---------------------------------------------------------------------------
# SPEC entry points
# ---------------------------------------------------------------------------

def _leaves_for(m: int, n: int, leaf_rows: int) -> int:
    P = max(1, m // max(1, leaf_rows))
    while P > 1 and m // P < n:
        P -= 1
    return P


def split_leaves(m: int, n: int, P: int, min_chains: int | None = None,
                 min_rows: int = 512, fill: bool = False, narrow: bool = False) -> int:
    """GPU chains per leaf (a power of two) for a leaf count P.

    A leaf processed as 2^k equal chains whose R factors are combined by a
    binary tree is the paper's hybrid tree: the
    binary tree over P*2^k chains combines every leaf's chains in its first
    k levels.  Chains stay >= max(min_rows, 4n) rows.  Default: split until
    there is one chain per SM (``min_chains``, default the SM count).  With
    ``fill`` (R-only chain kernel) the split maximises the wave fill
    chains / (waves x SMs) instead; a further split must gain > 2% fill
    (measured: C3's per-GPU shard at 4 GPUs runs 10% faster as 2 chains per
    leaf; splitting R + Q or the narrow kernel's leaves only adds tree and
    per-chain overhead, tools/prof_split.py).  With ``narrow`` (R only, n <= 8:
    one warp per chain, 8 warps per SM) the split goes on until there are more
    chains than warp slots: the library then deals the rows to exactly one
    wave of warps (CAQR_TUNE_FUSE; C4's per-GPU shard at 8 GPUs, 1024 leaves of
    16384 rows, would otherwise run on 128 of the 148 SMs).
    """
    if min_chains is None:
        min_chains = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count

    def ok(k):
        return m // (P * 2 * k) >= max(min_rows, 4 * n)

    if narrow:
        k = 1
        while P * k <= 8 * min_chains and ok(k):
            k *= 2
        return k if P * k > 8 * min_chains else 1

    if not fill:
        k = 1
        while P * k < min_chains and ok(k):
            k *= 2
        return k

    def frac(k):
        c = P * k
        return c / (-(-c // min_chains) * min_chains)

    best_k, best = 1, frac(1)
    k = 1
    while ok(k) and P * k < 16 * min_chains:
        k *= 2
        if frac(k) > best + 0.02:
            best_k, best = k, frac(k)
    return best_k


def tsqr(A, leaf_rows: int = 8192, q: str = "none", tree: ReductionTree | None = None,
         device=None, counter=None, split: bool = True, stream: bool = True):
    """Convenience TSQR: returns R, (R, factor) or (R, Q).

    q = "none" (R only), "implicit" (R + TsqrFactor) or "explicit" (R + thin Q).
    Leaves follow BlockRowLayout(m, n, floor(m / leaf_rows)); with ``split``
    (default, binary tree only) each leaf runs as 2^k GPU chains when there
    are fewer leaves than SMs (``split_leaves``).  R follows the reference's
    sign convention (beta = -sign(x0)||x||: mixed-sign diagonal).  A host
    matrix with q = "none" on the binary tree is streamed through the GPU in
    row chunks with the copies overlapped (``stream.tsqr_stream``; same
    leaves and tree, bitwise-identical R as long as no call has more leaves
    than the GPU has CTA / warp slots -- beyond that the library deals the rows
    of a call to longer runs, CAQR_TUNE_FUSE, and the two paths agree to
    rounding); ``stream=False`` copies it whole.
    """
    if q not in ("none", "implicit", "explicit"):
        raise ValueError(f"q must be none / implicit / explicit, got {q!r}")
    host_in = isinstance(A, np.ndarray) or (isinstance(A, torch.Tensor) and not A.is_cuda)
    if stream and host_in and q == "none" and (tree is None or tree.shape == BINARY):
        from .stream import tsqr_stream

        Ah = A if isinstance(A, torch.Tensor) else np.asarray(A, dtype=np.float64)
        if Ah.ndim != 2:
            raise DimensionError(f"matrix must be 2-D, got ndim={Ah.ndim}")
        m, n = Ah.shape
        if m < n:
            raise DimensionError(f"need m >= n, got {m} x {n}")
        if n < 1 or n > MAX_N:
            raise DimensionError(f"GPU TSQR supports 1 <= n <= {MAX_N}, got n = {n}")
        if tree is not None:
            P = tree.P
        else:
            P = _leaves_for(m, n, leaf_rows)
            if split:
                P *= split_leaves(m, n, P, fill=n > 8)
        BlockRowLayout(m, n, P)  # raises DimensionError for short leaves
        R = tsqr_stream(Ah, P, device=device)
        if counter is not None:
            _, h0, ht = _lib.geometry(n)
            _count(counter, BlockRowLayout(m, n, P), n, h0, ht, P)
        return _out(R, True)
    At, host = to_device(A, device)
    m, n = At.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if tree is not None:
        P = tree.P
    else:
        P = _leaves_for(m, n, leaf_rows)
        if split:
            P *= split_leaves(m, n, P, fill=(n > 8 and q == "none"), narrow=(n <= 8 and q == "none"))
    f = factor_device(At, P, want_q=(q != "none"), tree=tree, counter=counter, host=host)
    if q == "none":
        return f.R_out()
    if q == "implicit":
        return f.R_out(), f
    return f.R_out(), _out(explicit_q_device(f), host)


def tsqr_parallel(executor, blocks, tree: ReductionTree | None = None, want_q: bool = True,
                  counter=None) -> TsqrFactor:
    """SPEC tsqr_parallel(executor, blocks per worker, tree).

    ``blocks`` are the P row blocks (numpy or torch), which must follow
    BlockRowLayout(m, n, P) -- e.g. ``partition_block_rows(A, P)``.  The
    executor is a ``DeviceExecutor`` (the GPU group); reduce mode leaves R at
    the root.  All-reduce mode returns the same R (replicated on the host side
    it is bitwise identical by construction).
    """
    if not blocks:
        raise DimensionError("need at least one block")
    ex = executor if isinstance(executor, DeviceExecutor) else DeviceExecutor()
    dev = ex.torch_device()
    parts, host = [], False
    for i, b in enumerate(blocks):
        t, h = to_device(b, dev, name=f"block {i}")
        parts.append(t)
        host |= h
    ncols = {p.shape[1] for p in parts}
    if len(ncols) != 1:
        raise DimensionError(f"blocks have mismatched column counts {sorted(ncols)}")
    A = torch.cat(parts, dim=0)
    P = len(parts)
    lay = BlockRowLayout(A.shape[0], A.shape[1], P)
    if tuple(p.shape[0] for p in parts) != lay.block_rows:
        raise DimensionError("blocks must follow BlockRowLayout(m, n, P) "
                             f"({lay.block_rows}), got {tuple(p.shape[0] for p in parts)}")
    tree = tree if tree is not None else ReductionTree(P=P, shape=BINARY)
    with torch.cuda.device(dev):
        f = factor_device(A, P, want_q=want_q, tree=tree, counter=counter, host=host)
    ex.census(tree, f.n)
    return f


def tsqr_explicit_q(factor: TsqrFactor):
    """Thin Q (m x n) with orthonormal columns."""
    from .sequential import SequentialTsqrFactor

    if isinstance(factor, SequentialTsqrFactor):
        return factor.explicit_q()
    return _out(explicit_q_device(factor), factor.host)


def tsqr_apply_q(factor: TsqrFactor, C, transpose: bool = False):
    """Q C (C with n or m rows) or Q^T C (C with m rows)."""
    from .sequential import SequentialTsqrFactor

    if isinstance(factor, SequentialTsqrFactor):
        return factor.apply_q(C, transpose)
    Ct, host = to_device(C, factor.R.device, name="C")
    return _out(apply_q_device(factor, Ct, transpose), host or factor.host)


# SPEC module tsqr also holds the sequential flat-tree driver
from .sequential import BlockStore, SequentialTsqrFactor, choose_P_sequential, tsqr_sequential  # noqa: E402,F401
