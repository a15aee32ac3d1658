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
        out[("rec", rank)] = (dict(rec.stages), rec.messages_received, rec.words_received)
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


def _local_apply(f, C, transpose):
    """Full (or thin) local Q of an oracle.tsqr_reference factor (test helper)."""
    import oracle

    C = C.numpy().copy()
    n, offs = f["n"], f["offs"]
    if transpose:
        for i, (Y, tau) in enumerate(f["leaves"]):
            C[offs[i]:offs[i + 1]] = oracle.apply_dense(Y, tau, C[offs[i]:offs[i + 1]], transpose=True)
        for (lvl, a, b, Yb, tau) in f["nodes"]:
            ta, tb = oracle.apply_stacked(Yb, tau, C[offs[a]:offs[a] + n], C[offs[b]:offs[b] + n],
                                          transpose=True)
            C[offs[a]:offs[a] + n], C[offs[b]:offs[b] + n] = ta, tb
        return torch.from_numpy(C)
    if C.shape[0] == n and offs[-1] != n:
        full = np.zeros((offs[-1], C.shape[1]))
        full[:n] = C
        C = full
    for (lvl, a, b, Yb, tau) in reversed(f["nodes"]):
        ta, tb = oracle.apply_stacked(Yb, tau, C[offs[a]:offs[a] + n], C[offs[b]:offs[b] + n])
        C[offs[a]:offs[a] + n], C[offs[b]:offs[b] + n] = ta, tb
    for i, (Y, tau) in enumerate(f["leaves"]):
        C[offs[i]:offs[i + 1]] = oracle.apply_dense(Y, tau, C[offs[i]:offs[i + 1]])
    return torch.from_numpy(C)


def _q_worker(rank, world, port, A, leaf_rows, Cfull, out):
    import oracle
    from paper_0809_2407_b200.counters import CommRecorder
    from paper_0809_2407_b200.dist import (cross_tree, shard_rows, sharded_apply_q,
                                           sharded_explicit_q)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n = A.shape
        lo, hi = shard_rows(m, world, rank)
        P = max(1, (hi - lo) // leaf_rows)
        f = oracle.tsqr_reference(A[lo:hi], P)

        def combine(Ra, Rb):
            Yb, tau, R = oracle.stacked_qr(Ra.numpy(), Rb.numpy())
            return torch.from_numpy(R), (Yb, tau)

        def apply_node(node, Ca, Cb, transpose):
            ta, tb = oracle.apply_stacked(node[0], node[1], Ca.numpy(), Cb.numpy(), transpose)
            return torch.from_numpy(ta), torch.from_numpy(tb)

        _, nodes = cross_tree(torch.from_numpy(f["R"]), combine)
        rec = CommRecorder()
        Q = sharded_explicit_q(f, nodes, n, _local_apply, apply_node, recorder=rec)
        C = torch.from_numpy(Cfull[lo:hi].copy())
        QtC = sharded_apply_q(f, nodes, C, n, _local_apply, apply_node, transpose=True)
        back = sharded_apply_q(f, nodes, QtC, n, _local_apply, apply_node, transpose=False)
        out[rank] = (Q.numpy(), QtC.numpy(), back.numpy(), rec.messages_received)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_cross_tree_q_gloo(world):
    """Q across ranks: explicit Q and Q^T C / Q (Q^T C) against the single-process
    oracle over the same binary tree (power-of-two leaves per rank)."""
    import oracle

    rng = np.random.Generator(np.random.Philox(10 + world))
    m, n, leaf = 2048, 12, 128
    A = rng.standard_normal((m, n))
    Cfull = rng.standard_normal((m, 3))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_q_worker, args=(world, _free_port(), A, leaf, Cfull, out), nprocs=world, join=True)
    Q = np.vstack([out[r][0] for r in range(world)])
    QtC = np.vstack([out[r][1] for r in range(world)])
    back = np.vstack([out[r][2] for r in range(world)])
    fref = oracle.tsqr_reference(A, m // leaf)
    Qref = oracle.tsqr_reference_q(fref)
    eps = oracle.EPS
    assert np.max(np.abs(Q - Qref)) <= 100 * eps
    assert oracle.orthogonality(Q) <= 10 * n * eps
    # Q^T C: its first n rows are Q_thin^T C; the rest is the complement
    assert np.max(np.abs(QtC[:n] - Qref.T @ Cfull)) <= 100 * n * eps * np.linalg.norm(Cfull, 2)
    assert np.linalg.norm(back - Cfull) <= 10 * n * eps * np.linalg.norm(Cfull)
    # down the tree: every non-root rank receives exactly one n x n block
    assert out[0][3] == 0 and all(out[r][3] == 1 for r in range(1, world))


@pytest.mark.parametrize("world", [2, 4])
def test_par_runtime_model_check_gloo(world):
    """the cross-GPU tree's recorded critical path matches
    Eq. (4.1): log2 P messages exactly, packed-triangle words (n+1)/n x n^2/2."""
    from paper_0809_2407_b200.counters import CommRecorder, par_runtime_model_check

    rng = np.random.Generator(np.random.Philox(world + 10))
    m, n = 4096, 16
    A = rng.standard_normal((m, n))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, A, 256, False, out), nprocs=world, join=True)
    recs = []
    for r in range(world):
        stages, mr, wr = out[("rec", r)]
        rec = CommRecorder(messages_received=mr, words_received=wr)
        rec.stages = stages
        recs.append(rec)
    rep = par_runtime_model_check(m, n, world, recs)
    assert rep["messages_ok"] and rep["messages"] == (world - 1).bit_length()
    assert rep["words_ok"] and rep["words_ratio"] == pytest.approx((n + 1) / n)


def test_par_runtime_model_check_examples():
    """SPEC examples: P = 1 -> 0 messages / 0 words; P = 4, n = 10 -> 55 words per
    stage vs the model's 50 (ratio 1.1); P = 16, n = 32 -> 4 messages."""
    from paper_0809_2407_b200.counters import CommRecorder, par_runtime_model_check

    rep = par_runtime_model_check(100, 8, 1, [CommRecorder()])
    assert rep["messages"] == 0 and rep["words"] == 0 and rep["messages_ok"] and rep["words_ok"]

    def tree_recorders(P, n):
        recs = [CommRecorder() for _ in range(P)]
        k = 1
        while (1 << (k - 1)) < P:
            for f in range(0, P, 1 << k):
                s = f + (1 << (k - 1))
                if s < P:
                    recs[s].record_send(n * (n + 1) // 2)
                    recs[f].record_recv(n * (n + 1) // 2, stage=(k, "R"))
            k += 1
        return recs

    rep = par_runtime_model_check(400, 10, 4, tree_recorders(4, 10))
    assert rep["messages"] == 2 and rep["words"] == 2 * 55
    assert rep["words_ratio"] == pytest.approx(1.1)
    rep = par_runtime_model_check(16 * 64, 32, 16, tree_recorders(16, 32))
    assert rep["messages"] == 4 and rep["messages_ok"] and rep["words_ok"]
    # a wrong census is flagged
    recs = tree_recorders(4, 10)
    recs[0].record_recv(55, stage=(9, "R"))
    assert not par_runtime_model_check(400, 10, 4, recs)["messages_ok"]
