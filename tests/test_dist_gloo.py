"""Multi-rank host logic of the cross-GPU tree (paper_0809_2407_b200.dist) on
CPU with the gloo backend, world sizes 2 and 4; the combine is injected
(oracle stacked QR), so no GPU is needed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, A, leaf_rows, all_reduce, out):
    import oracle
    from paper_0809_2407_b200.counters import CommRecorder
    from paper_0809_2407_b200.dist import cross_tree, shard_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n = A.shape
        lo, hi = shard_rows(m, world, rank)
        P = max(1, (hi - lo) // leaf_rows)
        R_loc = torch.from_numpy(oracle.tsqr_reference(A[lo:hi], P)["R"])

        def combine(Ra, Rb):
            Yb, tau, R = oracle.stacked_qr(Ra.numpy(), Rb.numpy())
            return torch.from_numpy(R), (Yb, tau)

        rec = CommRecorder()
        R, nodes = cross_tree(R_loc, combine, all_reduce=all_reduce, recorder=rec)
        out[rank] = (None if R is None else R.numpy(), len(nodes), rec.messages_received,
                     rec.words_received, rec.messages_sent)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,all_reduce", [(2, False), (4, False), (4, True)])
def test_cross_tree_gloo(world, all_reduce):
    import oracle

    rng = np.random.Generator(np.random.Philox(world))
    A = rng.standard_normal((4096, 16))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, A, 256, all_reduce, out), nprocs=world, join=True)
    # reduce mode: R on rank 0 only; all-reduce: bitwise identical everywhere
    R0 = out[0][0]
    Rref = oracle.tsqr_reference(A, 16)["R"]
    assert oracle.r_diff(R0, Rref) <= 1000 * oracle.EPS
    for r in range(1, world):
        if all_reduce:
            assert np.array_equal(out[r][0], R0)
        else:
            assert out[r][0] is None
    # Eq. 4.1: log2(world) messages of n(n+1)/2 words reach the root
    n = 16
    lv = int(np.log2(world))
    assert out[0][2] == lv and out[0][3] == lv * n * (n + 1) // 2
    assert sum(out[r][4] for r in range(world)) == world - 1
