"""Sequential flat-tree TSQR over a BlockStore (Algorithm 2):
the SPEC's examples, element-wise parity of every Y_0k / tau_0k with the
oracle's Algorithm 2 (geqr2 on A_0, tri_rect_qr on [R; A_k]), the store's
transfer counters and the on-disk layout."""

import numpy as np
import pytest

import oracle
from oracle import EPS

pytestmark = pytest.mark.gpu


def _philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def _oracle_alg2(A, P):
    offs = oracle.block_rows(A.shape[0], A.shape[1], P)
    Y, tau, R = oracle.geqr2(A[offs[0]:offs[1]])
    out = [(Y, tau)]
    for k in range(1, P):
        V, tau, R = oracle.tri_rect_qr(R, A[offs[k]:offs[k + 1]])
        out.append((V, tau))
    return out, R


def test_p1_is_qr_unblocked_bitwise():
    from paper_0809_2407_b200.householder import qr_unblocked
    from paper_0809_2407_b200.sequential import BlockStore, tsqr_sequential

    A = _philox(1).standard_normal((64, 8))
    f = tsqr_sequential(BlockStore.from_matrix(A, 1))
    assert np.array_equal(f.R, qr_unblocked(A)[1])


@pytest.mark.parametrize("m,n,P,disk", [(64, 8, 4, False), (64, 8, 4, True), (5000, 40, 7, True),
                                        (1200, 150, 3, False)])
def test_sequential_parity_and_counters(m, n, P, disk, tmp_path):
    from paper_0809_2407_b200.sequential import BlockStore
    from paper_0809_2407_b200.tsqr import tsqr_apply_q, tsqr_explicit_q, tsqr_sequential

    A = _philox(m + n + P).standard_normal((m, n))
    st = BlockStore.from_matrix(A, P, directory=str(tmp_path / "s") if disk else None)
    f = tsqr_sequential(st)
    # SPEC example: R equals the dense-QR oracle's R up to signs, <= 1e-13 relative
    assert oracle.r_diff(f.R, np.linalg.qr(A, mode="r")) <= 1e-13
    # every stored chain factor matches the oracle's Algorithm 2 element-wise
    facs, Ro = _oracle_alg2(A, P)
    assert np.max(np.abs(f.R - Ro)) <= 100 * EPS * np.abs(Ro).max()
    for k, (Yo, to) in enumerate(facs):
        Y, tau = st.read_factor(k)
        assert np.max(np.abs(Y - Yo)) <= 1e-11 and np.max(np.abs(tau - to)) <= 1e-12
    # counters: each A block read once, each Y block written once
    c = st.counters()
    assert c["blocks_read"] == P and c["blocks_written"] == P
    assert c["words_read"] == m * n
    Q = tsqr_explicit_q(f)
    assert oracle.residual(A, Q, f.R) <= 10 * n * EPS and oracle.orthogonality(Q) <= 10 * n * EPS
    x = _philox(9).standard_normal((m, 2))
    assert np.max(np.abs(tsqr_apply_q(f, tsqr_apply_q(f, x, transpose=True)) - x)) <= 1e-12
    if disk:
        import os

        names = set(os.listdir(tmp_path / "s"))
        assert {"meta.json"} | {f"A_{k}.mat" for k in range(P)} | {f"Y_{k}.mat" for k in range(P)} \
            | {f"tau_{k}.vec" for k in range(P)} <= names
