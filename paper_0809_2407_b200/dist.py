"""Multi-GPU TSQR: 1-D block-row shards, one process per GPU.

Each rank factors its shard with the single-GPU path (local leaves + local
tree) and the per-rank R factors are then combined by the cross-GPU binary
tree of ``trees._binary`` over the ranks (PAPER.md:757-796 with P = world
size): at level k rank f + 2^(k-1) sends its packed R
(n(n+1)/2 doubles, the Eq. 4.1 message) to rank f, which runs the
stacked-triangle combine kernel.  Reduce mode leaves R on rank 0;
all-reduce mode broadcasts it back so every rank holds the bitwise-identical R.

Transport: ``torch.distributed`` point-to-point (NCCL over NVLink on GPUs,
gloo on CPU for the host-logic tests).  ``combine`` and ``local`` are
injectable so the host logic is testable without a GPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .trees import ReductionTree


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


def cross_tree(R_local: torch.Tensor, combine, group=None, all_reduce: bool = False,
               recorder=None):
    """Combine per-rank R factors up the binary tree over the ranks.

    ``combine(Ra, Rb) -> (R, node)`` runs on the receiver.  Returns (R or None,
    list of (level, partner, node) factors kept by this rank).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = R_local.shape[0]
    tree = ReductionTree(P=world)
    R = R_local
    nodes = []
    words = n * (n + 1) // 2
    for lvl, grp in enumerate(tree.levels, start=1):
        for (a, b) in grp:
            if rank == b:
                dist.send(pack_upper(R), dst=a, group=group)
                if recorder is not None:
                    recorder.record_send(words)
            elif rank == a:
                buf = torch.empty(words, dtype=R.dtype, device=R.device)
                dist.recv(buf, src=b, group=group)
                if recorder is not None:
                    recorder.record_recv(words, stage=(lvl, "R"))
                R, node = combine(R, unpack_upper(buf, n))
                nodes.append((lvl, b, node))
        # ranks that already sent are done with the factorization
    is_root = rank == tree.root
    if all_reduce:
        buf = pack_upper(R) if is_root else torch.empty(words, dtype=R.dtype, device=R.device)
        dist.broadcast(buf, src=tree.root, group=group)
        R = unpack_upper(buf, n)
        return R, nodes
    return (R if is_root else None), nodes


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
