"""Verifier arithmetic for parity tests (test oracle only).

``sign_normalize`` follows ``pkg/tests/oracles.py:14-18``.  Gram and
Frobenius sums are accumulated chunked-pairwise: a
naive Q^T Q over 10^8 rows shows a ~5 n eps defect on a correct Q.
"""

from __future__ import annotations

import numpy as np

EPS = float(np.finfo(np.float64).eps)


def sign_normalize(R):
    """Flip row signs so diag(R) >= 0 (oracles.py:14-18; 0 maps to +1)."""
    R = np.asarray(R, dtype=np.float64)
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return d[:, None] * R


def r_diff(R1, R2, scale=None):
    """max |sn(R1) - sn(R2)| / scale; scale defaults to sigma_max(R2)."""
    R1 = np.asarray(R1, dtype=np.float64)
    R2 = np.asarray(R2, dtype=np.float64)
    if scale is None:
        scale = float(np.linalg.svd(R2, compute_uv=False)[0]) or 1.0
    return float(np.max(np.abs(sign_normalize(R1) - sign_normalize(R2))) / scale)


def _pairwise_sum(parts):
    parts = list(parts)
    while len(parts) > 1:
        nxt = [parts[i] + parts[i + 1] for i in range(0, len(parts) - 1, 2)]
        if len(parts) % 2:
            nxt.append(parts[-1])
        parts = nxt
    return parts[0]


def gram_pairwise(Q, chunk=1 << 15):
    """Q^T Q with per-chunk BLAS products summed pairwise."""
    Q = np.asarray(Q)
    m = Q.shape[0]
    parts = []
    for s in range(0, m, chunk):
        blk = np.asarray(Q[s:s + chunk], dtype=np.float64)
        parts.append(blk.T @ blk)
    return _pairwise_sum(parts)


def orthogonality(Q, chunk=1 << 15):
    """||Q^T Q - I||_F (chunked-pairwise Gram)."""
    G = gram_pairwise(Q, chunk)
    return float(np.linalg.norm(G - np.eye(G.shape[0])))


def residual(A, Q, R, chunk=1 << 15):
    """||A - Q R||_F / ||A||_F, accumulated chunked-pairwise."""
    A = np.asarray(A)
    num, den = [], []
    for s in range(0, A.shape[0], chunk):
        a = np.asarray(A[s:s + chunk], dtype=np.float64)
        d = a - np.asarray(Q[s:s + chunk], dtype=np.float64) @ R
        num.append(float(np.sum(d * d)))
        den.append(float(np.sum(a * a)))
    return float(np.sqrt(_pairwise_sum(num)) / np.sqrt(_pairwise_sum(den)))
