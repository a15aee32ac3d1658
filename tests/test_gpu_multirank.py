"""The GPU kernels across ranks: 2 and 4 processes share cuda:0 and talk over
gloo (device tensors staged through host memory, paper_0809_2407_b200.dist
send / recv / broadcast), so no kernel waits on another rank's kernel.

* tsqr_sharded (dist.py): 1-D row shards, local TSQR on the GPU, the
  cross-rank binary tree of stacked-triangle combines (gpu_combine); R
  against LAPACK and the reference composition, the explicit Q gathered
  (residual, orthogonality), Q^T Q C = C through tsqr_sharded_apply_q, and
  all-reduce mode (every rank's R bitwise identical).
* caqr_grid (grid.py, Algorithm 3) with the GPU backend (GpuBackend pack /
  unpack / shapes, node factors received over the row broadcasts) on 2 x 2,
  2 x 1 and 1 x 2 grids; R against LAPACK and the reference's blocked QR.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)


def _gather_rows(t):
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, t.cpu().numpy())
    return np.vstack(parts)


def _tsqr_worker(rank, world, port, A, leaf, out):
    from paper_0809_2407_b200.dist import (shard_rows, tsqr_sharded, tsqr_sharded_apply_q,
                                           tsqr_sharded_explicit_q)

    _init(rank, world, port)
    try:
        m, n = A.shape
        lo, hi = shard_rows(m, world, rank)
        As = torch.from_numpy(A[lo:hi]).cuda()
        R, f, nodes = tsqr_sharded(As, leaf_rows=leaf, want_q=True)
        Q = _gather_rows(tsqr_sharded_explicit_q(f, nodes))
        C = torch.from_numpy(np.random.Generator(np.random.Philox(rank)).standard_normal((hi - lo, 3))).cuda()
        QtC = tsqr_sharded_apply_q(f, nodes, C, transpose=True)
        back = tsqr_sharded_apply_q(f, nodes, QtC, transpose=False)
        err = float(torch.max(torch.abs(back - C)))
        Rall, _, _ = tsqr_sharded(As, leaf_rows=leaf, all_reduce=True)
        Rs = [None] * world
        dist.all_gather_object(Rs, Rall.cpu().numpy())
        out[rank] = (None if R is None else R.cpu().numpy(), Q, err,
                     all(np.array_equal(Rs[0], x) for x in Rs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,leaf", [(2, 20000, 64, 2048), (4, 40000, 128, 4096),
                                            (4, 9000 + 7, 32, 1000), (2, 50000, 8, 4096)])
def test_tsqr_sharded_gpu_ranks(world, m, n, leaf):
    import oracle

    A = np.random.Generator(np.random.Philox(m + n)).standard_normal((m, n))
    out = mp.Manager().dict()
    mp.spawn(_tsqr_worker, args=(world, _free_port(), A, leaf, out), nprocs=world, join=True)
    R, Q, _, _ = out[0]
    scale = np.linalg.norm(A, 2)
    assert np.array_equal(R, np.triu(R))
    assert oracle.r_diff(R, np.linalg.qr(A, mode="r"), scale) <= 1000 * oracle.EPS
    Rref = oracle.tsqr_reference(A, world)["R"]  # the reference composition over `world` blocks
    assert oracle.r_diff(R, Rref, scale) <= 1000 * oracle.EPS
    assert oracle.residual(A, Q, R) <= 10 * n * oracle.EPS
    assert oracle.orthogonality(Q) <= 10 * n * oracle.EPS
    for r in range(world):
        assert out[r][2] <= 1e-12  # Q (Q^T C) = C
        assert out[r][3]          # all-reduce: bitwise-identical R on every rank


def _grid_worker(rank, world, port, A, b, Pr, Pc, leaf, out):
    from paper_0809_2407_b200.core import BlockCyclicLayout
    from paper_0809_2407_b200.grid import GpuBackend, caqr_grid, gather_R, make_grid, scatter_local

    _init(rank, world, port)
    try:
        m, n = A.shape
        grid = make_grid(BlockCyclicLayout(m, n, b, Pr, Pc))
        local = scatter_local(torch.from_numpy(A).cuda(), grid)
        res = caqr_grid(local, grid, GpuBackend(leaf_rows=leaf))
        R = gather_R(res)
        out[rank] = None if R is None else R.cpu().numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,b,Pr,Pc,leaf", [(1024, 768, 128, 2, 2, 256), (1536, 512, 128, 2, 1, 512),
                                              (768, 768, 64, 1, 2, 256)])
def test_caqr_grid_gpu_ranks(m, n, b, Pr, Pc, leaf):
    import oracle

    A = np.random.Generator(np.random.Philox(m * 3 + n)).standard_normal((m, n))
    out = mp.Manager().dict()
    mp.spawn(_grid_worker, args=(Pr * Pc, _free_port(), A, b, Pr, Pc, leaf, out), nprocs=Pr * Pc,
             join=True)
    R = out[0]
    scale = np.linalg.norm(A, 2)
    assert np.array_equal(R, np.triu(R))
    assert oracle.r_diff(R, np.linalg.qr(A, mode="r"), scale) <= 1000 * oracle.EPS
    _, _, Rb = oracle.blocked_qr(A, b)
    assert oracle.r_diff(R, Rb, scale) <= 1000 * oracle.EPS
