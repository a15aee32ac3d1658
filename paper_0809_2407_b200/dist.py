"""Multi-GPU TSQR: 1-D block-row shards, one process per GPU.

Each rank factors its shard with the single-GPU path (local leaves + local
tree) and the per-rank R factors are then combined by the cross-GPU binary
tree of ``trees._binary`` over the ranks (PAPER.md:757-796 with P = world
size): at level k rank f + 2^(k-1) sends its packed R
(n(n+1)/2 doubles, the Eq. 4.1 message) to rank f, which runs the
stacked-triangle combine kernel.  Reduce mode leaves R on rank 0;
all-reduce mode broadcasts it back so every rank holds the bitwise-identical R.

Q across ranks: with Q = diag(Q_r) Q_cross,
Q C applies the cross tree top-down to each rank's top n rows and then the
local Q; Q^T C applies the local Q^T and then the cross tree bottom-up
(``cross_apply``).  Each tree event moves one n x k block to the receiver
and back; forming Q explicitly skips the upward message (the partner's
block is still zero on the way down).

Transport: ``torch.distributed`` point-to-point (NCCL over NVLink on GPUs;
gloo, with device tensors staged through host memory, for the host-logic
tests and for several ranks sharing one GPU).  ``combine`` and ``local`` are
injectable so the host logic is testable without a GPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .trees import ReductionTree


# ---------------------------------------------------------------------------
# transport: NCCL moves device tensors directly; gloo (the host-logic tests,
# and several ranks sharing one GPU) stages device tensors through host memory
# ---------------------------------------------------------------------------
def _staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and dist.get_backend(group) == "gloo"


def send(t: torch.Tensor, group=None, group_dst=None, dst=None) -> None:
    x = t.cpu() if _staged(t, group) else t
    if group_dst is not None:
        dist.send(x, group=group, group_dst=group_dst)
    else:
        dist.send(x, dst=dst, group=group)


def recv(t: torch.Tensor, group=None, group_src=None, src=None) -> None:
    x = torch.empty(t.shape, dtype=t.dtype) if _staged(t, group) else t
    if group_src is not None:
        dist.recv(x, group=group, group_src=group_src)
    else:
        dist.recv(x, src=src, group=group)
    if x is not t:
        t.copy_(x)


def broadcast(t: torch.Tensor, group=None, group_src=None) -> None:
    x = t.cpu() if _staged(t, group) else t
    dist.broadcast(x, group=group, group_src=group_src)
    if x is not t:
        t.copy_(x)


def pack_upper(R: torch.Tensor) -> torch.Tensor:
    n = R.shape[0]
    iu = torch.triu_indices(n, n, device=R.device)
    return R[iu[0], iu[1]].contiguous()


def unpack_upper(p: torch.Tensor, n: int) -> torch.Tensor:
    R = torch.zeros((n, n), dtype=p.dtype, device=p.device)
    iu = torch.triu_indices(n, n, device=p.device)
    R[iu[0], iu[1]] = p
    return R


def shard_rows(m: int, world: int, rank: int):
    """Rows [lo, hi) of rank's shard: BlockRowLayout(m, n, world) semantics."""
    base = m // world
    lo = rank * base
    hi = m if rank == world - 1 else lo + base
    return lo, hi


def _members(group, members):
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    mem = list(range(world)) if members is None else list(members)
    return mem, (mem.index(me) if me in mem else None)


def cross_tree(R_local: torch.Tensor, combine, group=None, all_reduce: bool = False,
               recorder=None, members=None):
    """Combine per-rank R factors up the binary tree over the ranks.

    ``combine(Ra, Rb) -> (R, node)`` runs on the receiver.  ``members`` (group
    ranks in tree order; default all, in rank order) lets a subset take part
    with any rank as the root (virtual index 0) -- CAQR's panel tree is rooted
    at the diagonal-block owner.  Returns (R or None, list of (level, partner,
    node) factors kept by this rank); non-members return (None, []).
    """
    mem, v = _members(group, members)
    if v is None:
        return None, []
    n = R_local.shape[0]
    tree = ReductionTree(P=len(mem))
    R = R_local
    nodes = []
    words = n * (n + 1) // 2
    for lvl, grp in enumerate(tree.levels, start=1):
        for (a, b) in grp:
            if v == b:
                send(pack_upper(R), group=group, group_dst=mem[a])
                if recorder is not None:
                    recorder.record_send(words)
            elif v == a:
                buf = torch.empty(words, dtype=R.dtype, device=R.device)
                recv(buf, group=group, group_src=mem[b])
                if recorder is not None:
                    recorder.record_recv(words, stage=(lvl, "R"))
                R, node = combine(R, unpack_upper(buf, n))
                nodes.append((lvl, b, node))
        # ranks that already sent are done with the factorization
    is_root = v == tree.root
    if all_reduce:
        if len(mem) != dist.get_world_size(group):
            raise ValueError("all-reduce mode needs every rank of the group")
        buf = pack_upper(R) if is_root else torch.empty(words, dtype=R.dtype, device=R.device)
        broadcast(buf, group=group, group_src=mem[tree.root])
        R = unpack_upper(buf, n)
        return R, nodes
    return (R if is_root else None), nodes


def cross_apply(nodes, C_top: torch.Tensor, apply_node, transpose: bool = False, group=None,
                zero_partner: bool = False, recorder=None, members=None) -> torch.Tensor:
    """Apply Q_cross (top-down) or Q_cross^T (bottom-up) of the cross-rank tree
    to this rank's top block C_top (n x k); ``nodes`` is this rank's list from
    ``cross_tree`` (same ``members``).  ``apply_node(node, Ca, Cb, transpose)
    -> (Ca, Cb)`` runs on the receiver of each event (apply_stacked semantics,
    householder.py:377-396).  ``zero_partner`` (top-down only): the partner's
    block is zero on arrival, so it is not sent (explicit-Q formation)."""
    mem, v = _members(group, members)
    if v is None:
        return C_top
    tree = ReductionTree(P=len(mem))
    levels = list(enumerate(tree.levels, start=1))
    if not transpose:
        levels = levels[::-1]
    skip_up = zero_partner and not transpose
    node_of = {(lvl, partner): node for (lvl, partner, node) in nodes}
    C = C_top.contiguous()
    words = C.numel()
    for lvl, grp in levels:
        for (a, b) in grp:
            if v == b:
                if not skip_up:
                    send(C, group=group, group_dst=mem[a])
                    if recorder is not None:
                        recorder.record_send(words)
                buf = torch.empty_like(C)
                recv(buf, group=group, group_src=mem[a])
                if recorder is not None:
                    recorder.record_recv(words, stage=(lvl, "Q"))
                C = buf
            elif v == a:
                if skip_up:
                    Cb = torch.zeros_like(C)
                else:
                    Cb = torch.empty_like(C)
                    recv(Cb, group=group, group_src=mem[b])
                    if recorder is not None:
                        recorder.record_recv(words, stage=(lvl, "Q"))
                C, Cb = apply_node(node_of[(lvl, b)], C, Cb, transpose)
                C = C.contiguous()
                send(Cb.contiguous(), group=group, group_dst=mem[b])
                if recorder is not None:
                    recorder.record_send(words)
    return C


def sharded_apply_q(local_factor, nodes, C_shard: torch.Tensor, n: int, local_apply, apply_node,
                    transpose: bool = False, group=None, recorder=None) -> torch.Tensor:
    """Q C or Q^T C for the row-sharded TSQR (C_shard = this rank's rows of C).
    ``local_apply(local_factor, C, transpose)`` applies the rank's local Q
    (C with m_loc rows: full Q; C with n rows and transpose False: thin Q)."""
    if transpose:
        C = local_apply(local_factor, C_shard, True)
        C = C.clone()
        C[:n] = cross_apply(nodes, C[:n].clone(), apply_node, True, group, recorder=recorder)
        return C
    C = C_shard.clone()
    C[:n] = cross_apply(nodes, C[:n].clone(), apply_node, False, group, recorder=recorder)
    return local_apply(local_factor, C, False)


def sharded_explicit_q(local_factor, nodes, n: int, local_apply, apply_node,
                       group=None, device=None, recorder=None) -> torch.Tensor:
    """This rank's rows of the thin Q (Q [I; 0])."""
    mem, v = _members(group, None)
    root = ReductionTree(P=len(mem)).root
    S = torch.eye(n, dtype=torch.float64, device=device) if v == root else \
        torch.zeros((n, n), dtype=torch.float64, device=device)
    S = cross_apply(nodes, S, apply_node, False, group, zero_partner=True, recorder=recorder)
    return local_apply(local_factor, S, False)  # thin: Q_local [S; 0]


def gpu_apply_node(node, Ca: torch.Tensor, Cb: torch.Tensor, transpose: bool):
    """Q or Q^T of one stacked-triangle node on [Ca; Cb] (tsqr_f64_tree_apply_level)."""
    from . import _lib
    from .tsqr import _ptr, _stream

    lib = _lib.load()
    Yn, tn = node
    n, k = Ca.shape
    C = torch.cat([Ca, Cb]).contiguous()
    ev = torch.tensor([[0, 1, 0]], dtype=torch.int32, device=C.device)
    _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(Yn), _ptr(tn), n, _ptr(ev), 1, _ptr(C), k, n, k,
                                             int(bool(transpose)), 0, _stream(C.device)),
               "tsqr_f64_tree_apply_level")
    return C[:n], C[n:]


def gpu_local_apply(f, C: torch.Tensor, transpose: bool) -> torch.Tensor:
    from .tsqr import apply_q_device

    return apply_q_device(f, C, transpose)


def gpu_combine(Ra: torch.Tensor, Rb: torch.Tensor):
    """Stacked-triangle combine on the GPU (tsqr_f64_tree_factor_level, one event)."""
    from . import _lib
    from .tsqr import _ptr, _stream

    lib = _lib.load()
    n = Ra.shape[0]
    slots = torch.stack([Ra, Rb]).contiguous()
    ev = torch.tensor([[0, 1, 0]], dtype=torch.int32, device=Ra.device)
    Yn = torch.zeros((1, n, n), dtype=torch.float64, device=Ra.device)
    tn = torch.zeros((1, n), dtype=torch.float64, device=Ra.device)
    _lib.check(lib.tsqr_f64_tree_factor_level(_ptr(slots), n, _ptr(ev), 1, _ptr(Yn), _ptr(tn),
                                              _stream(Ra.device)), "tsqr_f64_tree_factor_level")
    return slots[0], (Yn[0], tn[0])


def tsqr_sharded(A_shard: torch.Tensor, leaf_rows: int = 8192, want_q: bool = False,
                 group=None, all_reduce: bool = False):
    """Distributed TSQR of the row-sharded matrix; returns (R or None, local factor, nodes)."""
    from .tsqr import _leaves_for, factor_device

    m_loc, n = A_shard.shape
    P = _leaves_for(m_loc, n, leaf_rows)
    f = factor_device(A_shard, P, want_q=want_q)
    R, nodes = cross_tree(f.R, gpu_combine, group=group, all_reduce=all_reduce)
    return R, f, nodes


def tsqr_sharded_apply_q(f, nodes, C_shard: torch.Tensor, transpose: bool = False, group=None):
    """Q C / Q^T C on the GPU for a ``tsqr_sharded(..., want_q=True)`` factorization."""
    return sharded_apply_q(f, nodes, C_shard, f.n, gpu_local_apply, gpu_apply_node, transpose, group)


def tsqr_sharded_explicit_q(f, nodes, group=None) -> torch.Tensor:
    """This rank's rows of the thin Q of a ``tsqr_sharded(..., want_q=True)`` factorization."""
    return sharded_explicit_q(f, nodes, f.n, gpu_local_apply, gpu_apply_node, group,
                              device=f.R.device)
