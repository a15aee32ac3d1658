"""Tall chain tiles with kept factors (CAQR_TUNE_CHAIN_HT_128 = 64): the leaf
chain of n in (64, 128] folds 64 rows per TRI_ON_RECT step (k_leaf_tt<64, 1, true>)
and Q / Q^T run through k_tall_apply.  Same checks as the 16-row format: leaf
factors element-wise against the oracle running the same hybrid algorithm
(qr_unblocked dense tile + qr_triangle_on_rect tiles, householder.py:297-332),
explicit Q, Q^T C, Q C, and CAQR against the reference's qr_blocked."""
import numpy as np
import pytest
import torch

import oracle
from oracle.checks import EPS

pytestmark = pytest.mark.gpu


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


@pytest.fixture(autouse=True)
def tall():
    from paper_0809_2407_b200 import _lib

    _lib.tune(_lib.TUNE_CHAIN_HT[128], 64)
    yield
    _lib.reset_tuning()


def factor(A, P):
    from paper_0809_2407_b200.tsqr import factor_device

    return factor_device(torch.from_numpy(np.ascontiguousarray(A)).cuda(), P, want_q=True)


@pytest.mark.parametrize("m,n,P", [(2000, 128, 2), (777, 100, 1), (300, 128, 1), (4096, 72, 3),
                                   (129, 128, 1), (5000, 120, 4), (148 * 300 + 5, 128, 148)])
def test_tall_leaf_factors_match_oracle(m, n, P):
    from paper_0809_2407_b200 import _lib

    A = philox(m + n).standard_normal((m, n))
    _, h0, ht = _lib.geometry(n)
    assert ht == 64
    f = factor(A, P)
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    scale = np.linalg.norm(A, 2)
    assert np.max(np.abs(f.R.cpu().numpy() - ref["R"])) <= 200 * EPS * scale
    Y = f.Y.cpu().numpy()
    tau = f.tau.cpu().numpy()
    offs = ref["offs"]
    for i, tiles in enumerate(ref["leaves"]):
        bnds = oracle.tsqr.chain_tiles(offs[i + 1] - offs[i], h0, ht)
        for k, ((V, t), (s, e)) in enumerate(zip(tiles[1:], bnds[1:]), start=1):
            Vg = Y[offs[i] + s: offs[i] + e]
            assert np.max(np.abs(Vg - V)) <= 1e-9 * max(1.0, np.max(np.abs(V))), (i, k)
            assert np.max(np.abs(tau[i, k] - t)) <= 1e-12, (i, k)
        if i > 3:
            break


@pytest.mark.parametrize("m,n,P", [(2000, 128, 2), (999, 100, 3), (20000, 128, 8), (640, 96, 1)])
def test_tall_explicit_q_and_applies(m, n, P):
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device

    A = philox(7 * m + n).standard_normal((m, n))
    _, h0, ht = _lib.geometry(n)
    f = factor(A, P)
    Q = explicit_q_device(f).cpu().numpy()
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    assert np.max(np.abs(Q - oracle.tsqr_hybrid_q(ref))) <= 1e-11
    R = f.R.cpu().numpy()
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    # Q^T C (C = [A, random]): the first n rows of Q^T A are R, the rest vanish; Q (Q^T C) = C
    for k in (n + 37, 150, 5):
        C = np.concatenate([A, philox(k).standard_normal((m, k))], axis=1)[:, :max(k, 1)]
        Ct = torch.from_numpy(np.ascontiguousarray(C)).cuda()
        QtC = apply_q_device(f, Ct, transpose=True)
        back = apply_q_device(f, QtC, transpose=False).cpu().numpy()
        assert np.max(np.abs(back - C)) <= 100 * n * EPS * np.max(np.abs(C))
        kk = min(k, n)
        top = QtC.cpu().numpy()[:n, :kk]
        assert np.max(np.abs(top - R[:, :kk])) <= 200 * EPS * np.linalg.norm(A, 2)
    # thin Q C
    Cn = philox(3).standard_normal((n, 40))
    QC = apply_q_device(f, torch.from_numpy(Cn).cuda(), transpose=False).cpu().numpy()
    assert np.max(np.abs(QC - Q @ Cn)) <= 100 * n * EPS * np.max(np.abs(Cn)) * np.sqrt(n)


def test_tall_caqr_matches_reference_blocked_qr():
    from paper_0809_2407_b200.caqr import caqr_factor

    m = n = 1536
    A = philox(5).standard_normal((m, n))
    f = caqr_factor(torch.from_numpy(A).cuda(), b=128, leaf_rows=512)
    R = f.R
    R = R.cpu().numpy() if hasattr(R, "cpu") else np.asarray(R)
    Rl = np.linalg.qr(A, mode="r")
    assert oracle.r_diff(R, Rl, np.linalg.norm(A, 2)) <= 1000 * EPS


def test_tall_run_to_run_bitwise():
    A = philox(11).standard_normal((148 * 700, 128))
    f1, f2 = factor(A, 148), factor(A, 148)
    assert torch.equal(f1.R, f2.R) and torch.equal(f1.Y, f2.Y) and torch.equal(f1.tau, f2.tau)


# ---- the n in (64, 128] tree kernels (k_tree_factor_dmma128, k_tree_apply_cp), default format ----

@pytest.mark.parametrize("m,n,P", [(3000, 72, 5), (2600, 100, 2), (4000, 127, 3), (5000, 128, 7),
                                   (1300, 65, 4)])
def test_wide_tree_nodes_match_oracle(m, n, P):
    """Node factors (qr_stacked_triangles, householder.py:263-294) element-wise against the
    oracle, explicit Q, and Q^T C / Q C with a column count that is not a multiple of 8
    (partial warps of the column-parallel tree apply), both directions, zero partner included."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device, factor_device

    _lib.reset_tuning()  # default 16-row leaf format; the tree kernels are the same for both
    A = philox(m * 3 + n).standard_normal((m, n))
    _, h0, ht = _lib.geometry(n)
    f = factor_device(torch.from_numpy(A).cuda(), P, want_q=True)
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    nY, nt = f.node_Y.cpu().numpy(), f.node_tau.cpu().numpy()
    for e, (lvl, a, b, Yb, tn) in enumerate(ref["nodes"]):
        assert np.max(np.abs(nY[e] - Yb)) <= 1e-9, e
        assert np.max(np.abs(nt[e] - tn)) <= 1e-12, e
    Q = explicit_q_device(f).cpu().numpy()
    assert np.max(np.abs(Q - oracle.tsqr_hybrid_q(ref))) <= 1e-11
    R = f.R.cpu().numpy()
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    for k in (37, 131):
        C = philox(k).standard_normal((m, k))
        Ct = torch.from_numpy(C).cuda()
        QtC = apply_q_device(f, Ct, transpose=True)
        assert np.max(np.abs(QtC.cpu().numpy()[:n] - Q.T @ C)) <= 200 * n * EPS * np.max(np.abs(C))
        back = apply_q_device(f, QtC, transpose=False).cpu().numpy()
        assert np.max(np.abs(back - C)) <= 100 * n * EPS * np.max(np.abs(C))


@pytest.mark.parametrize("kind", ["kappa1e12", "zero_columns", "duplicate_columns", "zero_matrix"])
def test_wide_tsqr_degenerate_inputs(kind):
    """n = 128 with kept factors on degenerate inputs (tau = 0 reflectors, sigma = 0 columns,
    kappa = 1e12): the column-block tree factor, the column-parallel tree apply and the leaf
    kernels keep the reference's bars (residual, orthogonality <= 10 n eps; pkg/tests/
    test_householder.py:340-350)."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

    _lib.reset_tuning()
    m, n, P = 6000, 128, 6
    rng = philox(17)
    if kind == "kappa1e12":
        U, _ = np.linalg.qr(rng.standard_normal((m, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        A = (U * np.logspace(0, -12, n)) @ V.T
    elif kind == "zero_columns":
        A = rng.standard_normal((m, n))
        A[:, [0, 5, 64, 127]] = 0.0
    elif kind == "duplicate_columns":
        A = rng.standard_normal((m, n))
        A[:, 70:80] = A[:, 10:20]
    else:
        A = np.zeros((m, n))
    f = factor_device(torch.from_numpy(A).cuda(), P, want_q=True)
    Q = explicit_q_device(f).cpu().numpy()
    R = f.R.cpu().numpy()
    assert np.all(np.isfinite(Q)) and np.all(np.isfinite(R))
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    scale = max(np.linalg.norm(A), 1e-300)
    assert np.linalg.norm(A - Q @ R) <= 10 * n * EPS * scale + 0.0
    assert np.allclose(np.tril(R, -1), 0.0)
