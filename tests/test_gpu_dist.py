"""GPU pieces of the cross-GPU tree (paper_0809_2407_b200.dist): the node
combine / apply kernels against the oracle, and the sharded driver end to end
in a one-rank NCCL group (only one GPU is reachable; the multi-rank message
pattern is covered by tests/test_dist_gloo.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
from oracle import EPS

pytestmark = pytest.mark.gpu


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


@pytest.mark.parametrize("n", [8, 32, 64, 128])
def test_gpu_combine_and_apply_node_match_oracle(n):
    from paper_0809_2407_b200.dist import gpu_apply_node, gpu_combine

    Ra = np.triu(philox(n).standard_normal((n, n)))
    Rb = np.triu(philox(n + 1).standard_normal((n, n)))
    R, node = gpu_combine(torch.from_numpy(Ra).cuda(), torch.from_numpy(Rb).cuda())
    Yb, tau, Rh = oracle.stacked_qr(Ra, Rb)
    scale = np.linalg.norm(np.vstack([Ra, Rb]), 2)
    assert oracle.r_diff(R.cpu().numpy(), Rh, scale) <= 100 * EPS
    Ca = philox(7).standard_normal((n, 5))
    Cb = philox(8).standard_normal((n, 5))
    for tr in (False, True):
        ga, gb = gpu_apply_node(node, torch.from_numpy(Ca).cuda(), torch.from_numpy(Cb).cuda(), tr)
        # the kernel's node carries its own signs: compare through the round trip
        # and against the oracle only where the reflectors agree (same algorithm)
        ha, hb = oracle.apply_stacked(Yb, tau, Ca, Cb, transpose=tr)
        got = np.vstack([ga.cpu().numpy(), gb.cpu().numpy()])
        assert np.max(np.abs(got - np.vstack([ha, hb]))) <= 1000 * EPS * np.linalg.norm(Ca) * 2
    ga, gb = gpu_apply_node(node, torch.from_numpy(Ca).cuda(), torch.from_numpy(Cb).cuda(), True)
    ba, bb = gpu_apply_node(node, ga, gb, False)
    assert np.max(np.abs(ba.cpu().numpy() - Ca)) <= 100 * n * EPS * np.linalg.norm(Ca)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_driver_one_rank_nccl():
    from paper_0809_2407_b200.dist import (tsqr_sharded, tsqr_sharded_apply_q,
                                           tsqr_sharded_explicit_q)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        A = torch.from_numpy(philox(3).standard_normal((16384, 64))).cuda()
        R, f, nodes = tsqr_sharded(A, leaf_rows=2048, want_q=True)
        Rh = np.linalg.qr(A.cpu().numpy(), mode="r")
        assert oracle.r_diff(R.cpu().numpy(), Rh) <= 1000 * EPS
        Q = tsqr_sharded_explicit_q(f, nodes).cpu().numpy()
        assert oracle.orthogonality(Q) <= 10 * 64 * EPS
        assert oracle.residual(A.cpu().numpy(), Q, R.cpu().numpy()) <= 10 * 64 * EPS
        C = torch.from_numpy(philox(4).standard_normal((16384, 3))).cuda()
        back = tsqr_sharded_apply_q(f, nodes, tsqr_sharded_apply_q(f, nodes, C, transpose=True))
        assert float(torch.linalg.norm(back - C)) <= 10 * 64 * EPS * float(torch.linalg.norm(C))
    finally:
        dist.destroy_process_group()
