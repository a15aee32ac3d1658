"""GPU backend of grid CAQR (paper_0809_2407_b200.grid): the broadcast payload
round trip and a 1 x 1 grid end to end under NCCL (one GPU reachable)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
from oracle import EPS

pytestmark = pytest.mark.gpu


def test_gpu_backend_pack_unpack_round_trip():
    from paper_0809_2407_b200.grid import GpuBackend

    be = GpuBackend(leaf_rows=512)
    piece = torch.from_numpy(np.random.default_rng(1).standard_normal((3072, 128))).cuda()
    f, R = be.local_factor(piece)
    Rb = torch.triu(torch.from_numpy(np.random.default_rng(2).standard_normal((128, 128)))).cuda()
    Rc, node = be.combine(R, Rb)
    keys = [(1, 1)]
    ts = be.pack(f, [(1, 1, node)])
    assert [tuple(t.shape) for t in ts] == [tuple(s) for s in be.shapes(3072, 128, keys)]
    f2, nodes2 = be.unpack([t.clone() for t in ts], 3072, 128, keys)
    C = torch.from_numpy(np.random.default_rng(3).standard_normal((3072, 40))).cuda()
    assert torch.equal(be.local_apply(f, C, True), be.local_apply(f2, C, True))
    a1, b1 = be.apply_node(node, C[:128], C[128:256], True)
    a2, b2 = be.apply_node(nodes2[0][2], C[:128], C[128:256], True)
    assert torch.equal(a1, a2) and torch.equal(b1, b2)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_grid_1x1_nccl_matches_lapack():
    from paper_0809_2407_b200.core import BlockCyclicLayout
    from paper_0809_2407_b200.grid import GpuBackend, caqr_grid, gather_R, make_grid, scatter_local

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        A = np.random.default_rng(4).standard_normal((1024, 512))
        grid = make_grid(BlockCyclicLayout(1024, 512, 128, 1, 1))
        local = scatter_local(torch.from_numpy(A).cuda(), grid)
        R = gather_R(caqr_grid(local, grid, GpuBackend(leaf_rows=256))).cpu().numpy()
        assert oracle.r_diff(R, np.linalg.qr(A, mode="r"), np.linalg.norm(A, 2)) <= 1000 * EPS
    finally:
        dist.destroy_process_group()
