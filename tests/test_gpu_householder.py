"""Kernel-level API (reference householder.py signatures) on the GPU against
the reference's golden outputs and known answers (pkg/tests/test_householder.py)."""

import numpy as np
import pytest

import oracle
from oracle import EPS

pytestmark = pytest.mark.gpu


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def test_house_gen_known_answers():
    from paper_0809_2407_b200.householder import house_gen

    v, t, b = house_gen(np.array([2.5, 0.0, 0.0]))
    assert t == 0.0 and b == 2.5
    v, t, b = house_gen(np.array([3.0, 4.0]))
    assert b == -5.0 and np.allclose(v, [1.0, 0.5]) and abs(t - 1.6) < 1e-15
    v, t, b = house_gen(np.zeros(2))
    assert t == 0.0 and b == 0.0
    v, t, b = house_gen(np.array([-3.0, 0.0]))
    assert b == 3.0 and t == 2.0
    for seed in range(20):
        x = philox(seed).uniform(-1e6, 1e6, 1 + seed % 12)
        v, t, b = house_gen(x)
        assert v[0] == 1.0
        assert abs(t * (2.0 - t * (v @ v))) <= 1e-13 * max(1.0, abs(t))
        y = x - t * v * (v @ x)
        sc = np.linalg.norm(x)
        assert abs(y[0] - b) <= 1e-13 * max(1.0, sc) and np.all(np.abs(y[1:]) <= 1e-13 * max(1.0, sc))


def test_unblocked_against_golden(golden):
    from paper_0809_2407_b200.householder import explicit_q, qr_unblocked

    g = golden["kernels"]
    for tag in ("unb_6x3", "unb_40x8", "unb_96x32"):
        A = g[f"{tag}_A"]
        f, R = qr_unblocked(A)
        assert np.max(np.abs(R - g[f"{tag}_R"])) <= 100 * EPS * np.abs(g[f"{tag}_R"]).max()
        assert np.max(np.abs(f.Y - g[f"{tag}_Y"])) <= 1e-12
        assert np.max(np.abs(f.tau - g[f"{tag}_tau"])) <= 1e-13
        assert np.max(np.abs(explicit_q(f) - g[f"{tag}_Q"])) <= 1e-12
    # taller than one block: the general geqr2 kernel, a DENSE factor with the
    # reference's own reflectors
    A = g["unb_160x64_A"]
    f, R = qr_unblocked(A)
    assert f.shape_tag == "dense"
    assert oracle.r_diff(R, g["unb_160x64_R"]) <= 100 * EPS
    assert np.max(np.abs(f.Y - g["unb_160x64_Y"])) <= 1e-12
    assert np.max(np.abs(f.tau - g["unb_160x64_tau"])) <= 1e-13
    Q = explicit_q(f)
    assert np.max(np.abs(Q - g["unb_160x64_Q"])) <= 1e-12
    assert oracle.residual(A, Q, R) <= 10 * 64 * EPS


def test_unblocked_known_answers():
    from paper_0809_2407_b200.householder import explicit_q, qr_unblocked

    f, R = qr_unblocked(np.eye(4))
    assert np.array_equal(R, np.eye(4)) and np.all(f.tau == 0.0)
    assert np.array_equal(explicit_q(qr_unblocked(np.eye(5))[0]), np.eye(5))
    A = np.triu(philox(3).standard_normal((5, 5)))
    np.fill_diagonal(A, np.abs(np.diag(A)) + 1.0)
    f, R = qr_unblocked(A)
    assert np.array_equal(R, A) and np.all(f.tau == 0.0)
    from paper_0809_2407_b200.core import DimensionError

    with pytest.raises(DimensionError):
        qr_unblocked(np.ones((2, 3)))


def test_stacked_against_golden(golden):
    from paper_0809_2407_b200.householder import apply_q, apply_qt, qr_stacked_triangles

    g = golden["kernels"]
    for n in (5, 8, 32, 64):
        tag = f"stk_{n}"
        f, R = qr_stacked_triangles([g[f"{tag}_Ra"], g[f"{tag}_Rb"]])
        assert np.max(np.abs(R - g[f"{tag}_R"])) <= 1e-12
        assert np.array_equal(f.Y[:n], np.eye(n))
        assert np.all(np.tril(f.Y[n:], -1) == 0.0)
        assert np.max(np.abs(f.Y - g[f"{tag}_Y"])) <= 1e-11
        assert np.max(np.abs(f.tau - g[f"{tag}_tau"])) <= 1e-13
        C = g[f"{tag}_C"]
        assert np.max(np.abs(apply_q(f, C) - g[f"{tag}_QC"])) <= 1e-12
        assert np.max(np.abs(apply_qt(f, C) - g[f"{tag}_QtC"])) <= 1e-12
    f, R = qr_stacked_triangles([np.eye(4), np.zeros((4, 4))])
    assert np.array_equal(R, np.eye(4)) and np.all(f.tau == 0.0)
    # three stacked triangles (test_householder.py:216-221)
    tris = [np.triu(philox(33 + i).standard_normal((4, 4))) for i in range(3)]
    f, R = qr_stacked_triangles(tris)
    _, _, Rd = oracle.geqr2(np.vstack(tris))
    assert np.max(np.abs(oracle.sign_normalize(R) - oracle.sign_normalize(Rd))) <= 1e-13
    from paper_0809_2407_b200.core import DimensionError

    with pytest.raises(DimensionError):
        qr_stacked_triangles([np.ones((3, 3)), np.eye(3)])


def test_triangle_on_rect_against_golden(golden):
    from paper_0809_2407_b200.householder import (apply_q, apply_qt, apply_qt_structured,
                                                  factor_t, qr_triangle_on_rect)

    g = golden["kernels"]
    for tag in ("tor_5x7", "tor_8x16", "tor_32x32", "tor_64x40"):
        f, R = qr_triangle_on_rect(g[f"{tag}_R0"], g[f"{tag}_B"])
        assert np.max(np.abs(R - g[f"{tag}_R"])) <= 1e-12
        assert np.max(np.abs(f.Y - g[f"{tag}_Y"])) <= 1e-11
        assert np.max(np.abs(f.tau - g[f"{tag}_tau"])) <= 1e-13
        C = g[f"{tag}_C"]
        assert np.max(np.abs(apply_q(f, C) - g[f"{tag}_QC"])) <= 1e-12
        assert np.max(np.abs(apply_qt(f, C) - g[f"{tag}_QtC"])) <= 1e-12
        T = factor_t(f)
        assert np.max(np.abs(T - g[f"{tag}_T"])) <= 1e-11
        n = R.shape[0]
        S0, S1 = apply_qt_structured(f, T, C[:n], C[n:])
        assert np.max(np.abs(S0 - g[f"{tag}_S0"])) <= 1e-12
        assert np.max(np.abs(S1 - g[f"{tag}_S1"])) <= 1e-12
    R = np.triu(philox(40).standard_normal((4, 4)))
    np.fill_diagonal(R, np.abs(np.diag(R)) + 0.5)
    f, R2 = qr_triangle_on_rect(R, np.zeros((3, 4)))
    assert np.array_equal(R2, R) and np.all(f.tau == 0.0)


def test_blocked_against_golden(golden):
    """qr_blocked keeps the reference's DENSE factor (geqr2 reflectors, tau)."""
    from paper_0809_2407_b200.householder import qr_blocked

    g = golden["kernels"]
    f, R = qr_blocked(g["blk_256x128_A"], 32)
    assert f.shape_tag == "dense"
    assert oracle.r_diff(R, g["blk_256x128_R"]) <= 1000 * EPS
    assert np.max(np.abs(f.tau - g["blk_256x128_tau"])) <= 1e-12


def test_general_shapes_beyond_one_block():
    """No shape limit beyond the reference's (householder.py:89-332): the general
    geqr2 kernel covers house_gen L > 128, qr_unblocked n > 128, stacked factors
    with (q-1) n > 128 and triangle-on-rectangle with r > 128, checked against
    the oracle restatement element by element."""
    from paper_0809_2407_b200.householder import (apply_q, explicit_q, house_gen,
                                                  qr_stacked_triangles, qr_triangle_on_rect,
                                                  qr_unblocked)

    x = philox(50).standard_normal(1000)
    v, tau, beta = house_gen(x)
    vo, to, bo = oracle.reflector(x)
    assert abs(beta - bo) <= 4 * EPS * abs(bo) and abs(tau - to) <= 4 * EPS
    assert np.max(np.abs(v - vo)) <= 1e-13
    A = philox(51).standard_normal((300, 150))
    f, R = qr_unblocked(A)
    Yo, to, Ro = oracle.geqr2(A)
    assert np.max(np.abs(R - Ro)) <= 100 * EPS * np.abs(Ro).max()
    assert np.max(np.abs(f.Y - Yo)) <= 1e-11 and np.max(np.abs(f.tau - to)) <= 1e-12
    Q = explicit_q(f)
    assert oracle.residual(A, Q, R) <= 10 * 150 * EPS and oracle.orthogonality(Q) <= 10 * 150 * EPS
    C = philox(52).standard_normal((300, 7))
    assert np.max(np.abs(apply_q(f, apply_q(f, C), transpose=True) - C)) <= 1e-12
    # q = 3 stacked triangles, n = 80: dense geqr2 of the stack keeps the profile
    rng = philox(53)
    Rs = [np.triu(rng.standard_normal((80, 80))) for _ in range(3)]
    fs, Rst = qr_stacked_triangles(Rs)
    S = np.vstack(Rs)
    assert oracle.r_diff(Rst, np.linalg.qr(S, mode="r")) <= 100 * EPS
    prof = np.zeros_like(fs.Y, dtype=bool)
    for j in range(80):
        prof[fs.reflector(j)[0], j] = True
    assert np.all(fs.Y[~prof] == 0.0) and np.array_equal(fs.Y[:80], np.eye(80))
    Qs = explicit_q(fs)
    assert oracle.residual(S, Qs, Rst) <= 10 * 80 * EPS
    # triangle on a 200-row rectangle
    R0 = np.triu(rng.standard_normal((70, 70)))
    B = rng.standard_normal((200, 70))
    ft, Rt = qr_triangle_on_rect(R0, B)
    Vo, tauo, Rto = oracle.tri_rect_qr(R0, B)
    assert np.max(np.abs(Rt - Rto)) <= 100 * EPS * np.abs(Rto).max()
    assert np.max(np.abs(ft.Y - Vo)) <= 1e-12 and np.max(np.abs(ft.tau - tauo)) <= 1e-13


def test_blocked_recursive_bitwise_relations():
    """The reference's own structural identities (test_householder.py:98-128):
    qr_blocked(nb = 1) IS qr_unblocked, qr_recursive without a split IS
    qr_blocked(nb = n) -- bitwise, on one block and beyond it."""
    from paper_0809_2407_b200.householder import qr_blocked, qr_recursive, qr_unblocked

    for (m, n) in [(16, 6), (20, 6), (400, 140)]:
        A = philox(60 + m).standard_normal((m, n))
        _, R1 = qr_unblocked(A)
        _, R2 = qr_blocked(A, nb=1)
        assert np.array_equal(R1, R2)
        _, R3 = qr_blocked(A, nb=n)
        _, R4 = qr_recursive(A, min_width=n)
        assert np.array_equal(R3, R4) and np.array_equal(R1, R3)


def test_recursive_elmroth_gustavson():
    """qr_recursive splits columns in halves and merges T (householder.py:214-251):
    R against the oracle, the cached T reproduces Q = I - Y T Y^T."""
    from paper_0809_2407_b200.householder import explicit_q, form_t, qr_recursive

    for (m, n, mw) in [(32, 8, 2), (300, 130, 16), (64, 33, 1)]:
        A = philox(70 + n).standard_normal((m, n))
        f, R = qr_recursive(A, min_width=mw)
        Ro = oracle.geqr2(A)[2]
        assert oracle.r_diff(R, Ro) <= 100 * EPS
        Y = f.Y
        Qt = np.eye(m)[:, :n] - Y @ (f.T @ (Y[:n].T))
        Q = explicit_q(f)
        assert np.max(np.abs(Q - Qt)) <= 1e-12
        assert oracle.residual(A, Q, R) <= 10 * n * EPS
        assert np.max(np.abs(form_t(Y, f.tau) - f.T)) <= 1e-12 * max(1.0, np.abs(f.T).max())


def test_form_t_kernel_against_oracle():
    """form_t (householder.py:148-164): the device recurrence equals the oracle's
    larft, including tau = 0 columns (the recurrence is skipped there)."""
    from paper_0809_2407_b200.householder import form_t

    Y, tau, _ = oracle.geqr2(philox(80).standard_normal((300, 40)))
    tau = tau.copy()
    tau[[3, 17]] = 0.0
    T = form_t(Y, tau)
    To = oracle.larft(Y, tau)
    assert np.max(np.abs(T - To)) <= 1e-13 * np.abs(To).max()
    assert np.all(T[:4, 3] == 0.0) and np.all(T[:18, 17] == 0.0)
