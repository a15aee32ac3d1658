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
    # taller than one block: CHAIN factor, same R up to rounding
    A = g["unb_160x64_A"]
    f, R = qr_unblocked(A)
    assert f.shape_tag == "chain"
    assert oracle.r_diff(R, g["unb_160x64_R"]) <= 100 * EPS
    Q = explicit_q(f)
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


def test_blocked_is_caqr(golden):
    from paper_0809_2407_b200.householder import qr_blocked

    g = golden["kernels"]
    f, R = qr_blocked(g["blk_256x128_A"], 32)
    assert oracle.r_diff(R, g["blk_256x128_R"]) <= 1000 * EPS
