"""Pin the CPU oracle: golden vectors produced by the reference itself
(oracle/make_golden.py) and the reference's own known-answer tests."""

import numpy as np
import pytest

import oracle
from oracle import EPS

TIGHT = 64 * EPS  # restatement vs reference: same operations, last-ulp slack


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1.0, np.max(np.abs(b))))


# ---- reference known answers (pkg/tests/test_householder.py) ---------------

def test_house_gen_known_answers():
    # test_householder.py:28-50
    v, t, b = oracle.reflector(np.array([2.5, 0.0, 0.0]))
    assert t == 0.0 and b == 2.5
    v, t, b = oracle.reflector(np.array([3.0, 4.0]))
    assert b == -5.0 and np.allclose(v, [1.0, 0.5]) and abs(t - 1.6) < 1e-15
    v, t, b = oracle.reflector(np.zeros(2))
    assert t == 0.0 and b == 0.0
    v, t, b = oracle.reflector(np.array([-3.0, 0.0]))
    assert b == 3.0 and t == 2.0


def test_identity_and_triangular_bitwise():
    # test_householder.py:68-79
    Y, tau, R = oracle.geqr2(np.eye(4))
    assert np.array_equal(R, np.eye(4)) and np.all(tau == 0.0)
    A = np.triu(np.random.Generator(np.random.Philox(3)).standard_normal((5, 5)))
    np.fill_diagonal(A, np.abs(np.diag(A)) + 1.0)
    Y, tau, R = oracle.geqr2(A)
    assert np.array_equal(R, A) and np.all(tau == 0.0)


def test_stacked_identity_over_zero():
    # test_householder.py:160-163
    Yb, tau, R = oracle.stacked_qr(np.eye(4), np.zeros((4, 4)))
    assert np.array_equal(R, np.eye(4)) and np.all(tau == 0.0)


def test_tri_rect_zero_rectangle_bitwise():
    # test_householder.py:225-231
    R = np.triu(np.random.Generator(np.random.Philox(40)).standard_normal((4, 4)))
    np.fill_diagonal(R, np.abs(np.diag(R)) + 0.5)
    V, tau, R2 = oracle.tri_rect_qr(R, np.zeros((3, 4)))
    assert np.array_equal(R2, R) and np.all(tau == 0.0)


def test_rejections():
    with pytest.raises(oracle.DimensionError):
        oracle.geqr2(np.ones((2, 3)))
    with pytest.raises(oracle.DimensionError):
        oracle.stacked_qr(np.ones((3, 3)), np.eye(3))
    with pytest.raises(oracle.DimensionError):
        oracle.tri_rect_qr(np.eye(3), np.ones((2, 4)))
    with pytest.raises(ValueError):
        oracle.geqr2(np.array([[1.0, np.nan], [0.0, 1.0]]))


# ---- golden vectors from the reference -------------------------------------

def _cases(g, prefix):
    return sorted({k.rsplit("_", 1)[0] for k in g if k.startswith(prefix)})


def test_geqr2_matches_reference(golden):
    g = golden["kernels"]
    tags = _cases(g, "unb_")
    assert len(tags) == 4
    for tag in tags:
        Y, tau, R = oracle.geqr2(g[f"{tag}_A"])
        assert rel(R, g[f"{tag}_R"]) <= TIGHT, tag
        assert rel(Y, g[f"{tag}_Y"]) <= TIGHT, tag
        assert rel(tau, g[f"{tag}_tau"]) <= TIGHT, tag
        assert rel(oracle.larft(Y, tau), g[f"{tag}_T"]) <= TIGHT, tag
        m, n = g[f"{tag}_A"].shape
        E = np.zeros((m, n))
        E[:n] = np.eye(n)
        assert rel(oracle.apply_dense(Y, tau, E), g[f"{tag}_Q"]) <= TIGHT, tag


def test_stacked_matches_reference(golden):
    g = golden["kernels"]
    for tag in _cases(g, "stk_"):
        Yb, tau, R = oracle.stacked_qr(g[f"{tag}_Ra"], g[f"{tag}_Rb"])
        n = Yb.shape[0]
        Yref = g[f"{tag}_Y"]
        assert np.array_equal(Yref[:n], np.eye(n)), tag
        assert rel(Yb, Yref[n:]) <= TIGHT, tag
        assert rel(tau, g[f"{tag}_tau"]) <= TIGHT, tag
        assert rel(R, g[f"{tag}_R"]) <= TIGHT, tag
        C = g[f"{tag}_C"]
        top, bot = oracle.apply_stacked(Yb, tau, C[:n], C[n:])
        assert rel(np.vstack([top, bot]), g[f"{tag}_QC"]) <= TIGHT, tag
        top, bot = oracle.apply_stacked(Yb, tau, C[:n], C[n:], transpose=True)
        assert rel(np.vstack([top, bot]), g[f"{tag}_QtC"]) <= TIGHT, tag


def test_tri_rect_matches_reference(golden):
    g = golden["kernels"]
    for tag in _cases(g, "tor_"):
        V, tau, R = oracle.tri_rect_qr(g[f"{tag}_R0"], g[f"{tag}_B"])
        n = R.shape[0]
        assert rel(V, g[f"{tag}_Y"]) <= TIGHT, tag
        assert rel(tau, g[f"{tag}_tau"]) <= TIGHT, tag
        assert rel(R, g[f"{tag}_R"]) <= TIGHT, tag
        C = g[f"{tag}_C"]
        top, bot = oracle.apply_tri_rect(V, tau, C[:n], C[n:])
        assert rel(np.vstack([top, bot]), g[f"{tag}_QC"]) <= TIGHT, tag
        top, bot = oracle.apply_tri_rect(V, tau, C[:n], C[n:], transpose=True)
        assert rel(np.vstack([top, bot]), g[f"{tag}_QtC"]) <= TIGHT, tag
        # apply_qt_structured (householder.py:361-364) equals Q^T [C0; C1]
        assert rel(np.vstack([top, bot]), np.vstack([g[f"{tag}_S0"], g[f"{tag}_S1"]])) <= 1e-13


def test_blocked_matches_reference(golden):
    g = golden["kernels"]
    Y, tau, R = oracle.blocked_qr(g["blk_256x128_A"], 32)
    assert rel(R, g["blk_256x128_R"]) <= TIGHT
    assert rel(tau, g["blk_256x128_tau"]) <= TIGHT


def test_composed_tsqr_matches_reference(golden):
    g = golden["tsqr"]
    for tag in _cases(g, "tsqr_"):
        A = g[f"{tag}_A"]
        P = int(tag.split("_P")[1])
        f = oracle.tsqr_reference(A, P)
        assert list(f["offs"]) == list(g[f"{tag}_offs"])
        assert rel(f["R"], g[f"{tag}_R"]) <= TIGHT, tag
        Q = oracle.tsqr_reference_q(f)
        assert rel(Q, g[f"{tag}_Q"]) <= TIGHT, tag


def test_schedules_match_reference(golden):
    g = golden["misc"]
    for k, v in g.items():
        if not k.startswith("sched_"):
            continue
        P = int(k.split("_")[1])
        assert np.array_equal(np.array(oracle.binary_events(P), dtype=np.int64).reshape(-1, 3), v)


# ---- the hybrid (GPU-structured) composition against the reference ---------

@pytest.mark.parametrize("n,h0,ht", [(32, 256, 32), (64, 256, 32), (16, 256, 32), (128, 128, 16)])
def test_hybrid_tsqr_meets_tolerances(golden, n, h0, ht):
    rng = np.random.Generator(np.random.Philox(n))
    A = rng.standard_normal((3000, n))
    f = oracle.tsqr_hybrid(A, 3, h0, ht)
    Q = oracle.tsqr_hybrid_q(f)
    Rref = oracle.tsqr_reference(A, 3)["R"]
    assert oracle.r_diff(f["R"], Rref) <= 1000 * EPS
    assert oracle.residual(A, Q, f["R"]) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    # apply(Q^T) then apply(Q) round trip through the hybrid tree
    C = rng.standard_normal((3000, 3))
    back = oracle.tsqr.tsqr_hybrid_apply(f, oracle.tsqr.tsqr_hybrid_apply(f, C, True), False)
    assert np.max(np.abs(back - C)) <= 100 * n * EPS * np.linalg.norm(C)


def test_hybrid_ill_conditioned(golden):
    g = golden["tsqr"]
    A = g["tsqr_1024x64_P8_A"]  # kappa = 1e12
    f = oracle.tsqr_hybrid(A, 2, 256, 32)
    Q = oracle.tsqr_hybrid_q(f)
    n = 64
    assert oracle.r_diff(f["R"], g["tsqr_1024x64_P8_R"]) <= 1000 * EPS
    assert oracle.residual(A, Q, f["R"]) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS


def test_caqr_oracle_matches_blocked(golden):
    rng = np.random.Generator(np.random.Philox(5))
    A = rng.standard_normal((512, 384))
    R, panels = oracle.tsqr.caqr_tsqr(A, 128, 128, 128, 16)
    _, _, Rb = oracle.blocked_qr(A, 128)
    assert oracle.r_diff(R, Rb) <= 1000 * EPS
