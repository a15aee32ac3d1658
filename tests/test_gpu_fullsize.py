"""Parity at BASELINE's full sizes through size-independent properties (the CPU
oracle cannot run these sizes in a test): an orthogonal Q preserves column
norms and the Gram matrix, so R^T R = A^T A and ||R e_j|| = ||A e_j||; for
explicit Q, ||Q^T Q - I|| and ||A - QR|| directly.  Inputs are seeded
synthetic matrices with the configs' shapes and distributions."""

import numpy as np
import pytest
import torch

from oracle import EPS

pytestmark = pytest.mark.gpu


def _gram_checks(A, R, n):
    an = torch.linalg.vector_norm(A, dim=0)
    rn = torch.linalg.vector_norm(R, dim=0)
    assert float(torch.max(torch.abs(rn - an) / an)) <= 100 * n * EPS
    G = A.T @ A
    assert float(torch.linalg.matrix_norm(R.T @ R - G) / torch.linalg.matrix_norm(G)) <= 100 * n * EPS
    assert torch.equal(R, torch.triu(R))


def test_c3_full_size_r_only():
    """C3: 16777216 x 128 N(0,1), 2048 leaves of 8192 rows, R only (16 GiB)."""
    from paper_0809_2407_b200.tsqr import tsqr

    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(1 << 24, 128, dtype=torch.float64, device="cuda", generator=g)
    R = tsqr(A, leaf_rows=8192)
    _gram_checks(A, R, 128)


def test_c4_full_size_r_only():
    """C4: 134217728 x 8 U(-1, 1), 8192 leaves of 16384 rows (narrow kernel, 8 GiB)."""
    from paper_0809_2407_b200.tsqr import tsqr

    g = torch.Generator(device="cuda").manual_seed(4)
    A = torch.rand(1 << 27, 8, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    R = tsqr(A, leaf_rows=16384)
    _gram_checks(A, R, 8)


def test_c2_full_size_explicit_q_kappa_1e12():
    """C2: 1048576 x 64 with geometric singular values 1 .. 1e-12 (gen_cond_matrix's
    profile, core.py:155-162; U, V from QR of seeded Gaussians), R + explicit Q."""
    from paper_0809_2407_b200.tsqr import tsqr

    m, n = 1 << 20, 64
    g = torch.Generator(device="cuda").manual_seed(2)
    U, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g))
    V, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
    sig = torch.tensor(np.logspace(0, -12, n), dtype=torch.float64, device="cuda")
    A = (U * sig) @ V.T
    R, Q = tsqr(A, leaf_rows=4096, q="explicit")
    orth = float(torch.linalg.matrix_norm(Q.T @ Q - torch.eye(n, dtype=torch.float64, device="cuda")))
    assert orth <= 10 * n * EPS
    res = float(torch.linalg.matrix_norm(A - Q @ R) / torch.linalg.matrix_norm(A))
    assert res <= 10 * n * EPS
    assert torch.equal(R, torch.triu(R))
