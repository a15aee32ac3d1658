"""Competitors and the stability sweep on the GPU (module
alt-factorizations).

The point of the sweep is the paper's section 5 claim: Householder-based TSQR
is unconditionally stable, while CholeskyQR, CGS and MGS lose orthogonality
with the condition number (quadratically for CholeskyQR).  Every algorithm
runs on the GPU:

* cholesky_qr: Gram A^T A (one library GEMM), our own unblocked Cholesky with
  failure detection (``tsqr_f64_cholesky``), Q = A R^-1 (triangular solve);
* cgs / mgs_row: classical and row-oriented modified Gram-Schmidt, column by
  column (library GEMV / rank-1 updates);
* TSQR (binary tree, P leaves), TSQR flat (the sequential Algorithm 2 driver)
  and Householder (qr_unblocked) from this package's kernels.

``stability_sweep`` reports ||Q^T Q - I||_F and ||A - QR||_F / ||A||_F per
(algorithm, kappa), with failures recorded as outcome "failed" rather than
aborting the sweep.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import CondSpec, DimensionError, gen_cond_matrix
from .tsqr import _ptr, _stream

EPS = float(np.finfo(np.float64).eps)


class CholeskyFailure(ArithmeticError):
    """Gram matrix not numerically positive definite."""


def _dev(A):
    t = torch.as_tensor(np.asarray(A, dtype=np.float64) if not isinstance(A, torch.Tensor) else A,
                        dtype=torch.float64)
    return t.to("cuda").contiguous()


def cholesky_qr(A):
    """(Q, R) with R^T R = A^T A and Q = A R^-1."""
    At = _dev(A)
    m, n = At.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    lib = _lib.load()
    G = (At.T @ At).contiguous()
    info = torch.zeros(1, dtype=torch.int32, device=At.device)
    _lib.check(lib.tsqr_f64_cholesky(_ptr(G), n, n, _ptr(info), _stream(At.device)),
               "tsqr_f64_cholesky")
    if int(info.item()):
        raise CholeskyFailure(f"Gram matrix not numerically positive definite (pivot {int(info.item()) - 1})")
    R = torch.triu(G)
    Q = torch.linalg.solve_triangular(R, At, upper=True, left=False)
    return Q, R


def _rank_check(r, j):
    if not float(r) > 0.0:
        raise DimensionError(f"zero-norm pivot column {j}: numerically rank deficient")


def cgs(A):
    """Classical Gram-Schmidt."""
    At = _dev(A)
    m, n = At.shape
    Q = torch.zeros_like(At)
    R = torch.zeros((n, n), dtype=torch.float64, device=At.device)
    for j in range(n):
        v = At[:, j].clone()
        if j:
            R[:j, j] = Q[:, :j].T @ At[:, j]
            v -= Q[:, :j] @ R[:j, j]
        R[j, j] = torch.linalg.vector_norm(v)
        _rank_check(R[j, j], j)
        Q[:, j] = v / R[j, j]
    return Q, R


def mgs_row(A):
    """Row-oriented modified Gram-Schmidt: each new q_j is projected out of all
    remaining columns at once."""
    W = _dev(A).clone()
    m, n = W.shape
    Q = torch.zeros_like(W)
    R = torch.zeros((n, n), dtype=torch.float64, device=W.device)
    for j in range(n):
        R[j, j] = torch.linalg.vector_norm(W[:, j])
        _rank_check(R[j, j], j)
        Q[:, j] = W[:, j] / R[j, j]
        if j + 1 < n:
            R[j, j + 1:] = Q[:, j] @ W[:, j + 1:]
            W[:, j + 1:] -= torch.outer(Q[:, j], R[j, j + 1:])
    return Q, R


def _tsqr_binary(A, P):
    from .tsqr import explicit_q_device, factor_device

    f = factor_device(_dev(A), P, want_q=True)
    return explicit_q_device(f), f.R_out()


def _tsqr_flat(A, P):
    from .sequential import BlockStore, tsqr_sequential

    f = tsqr_sequential(BlockStore.from_matrix(np.asarray(A), P))
    return torch.as_tensor(f.explicit_q(), device="cuda"), torch.as_tensor(f.R, device="cuda")


def _householder(A):
    from .householder import explicit_q, qr_unblocked

    f, R = qr_unblocked(np.asarray(A))
    return torch.as_tensor(explicit_q(f), device="cuda"), torch.as_tensor(R, device="cuda")


def _measures(A, Q, R):
    At = _dev(A)
    n = At.shape[1]
    orth = float(torch.linalg.matrix_norm(Q.T @ Q - torch.eye(n, dtype=torch.float64, device=Q.device)))
    res = float(torch.linalg.matrix_norm(At - Q @ R) / torch.linalg.matrix_norm(At))
    return orth, res


@dataclass
class StabilityReport:
    """Rows of (algorithm, kappa, seed, orthogonality, residual, outcome)."""

    rows: list = field(default_factory=list)

    def cell(self, algorithm, kappa):
        return [r for r in self.rows if r[0] == algorithm and r[1] == kappa]


def stability_sweep(kappas, m: int = 1000, n: int = 50, seeds=1, P: int = 4) -> StabilityReport:
    """Every algorithm on gen_cond_matrix(CondSpec(m, n, kappa, seed)) for each
    kappa and seed; a failure becomes outcome "failed"."""
    algos = {
        f"TSQR(binary,P={P})": lambda A: _tsqr_binary(A, P),
        f"TSQR(flat,P={P})": lambda A: _tsqr_flat(A, P),
        "Householder": _householder,
        "CGS": cgs,
        "MGS": mgs_row,
        "CholeskyQR": cholesky_qr,
    }
    rep = StabilityReport()
    seed_list = range(seeds) if isinstance(seeds, int) else list(seeds)
    for kappa in kappas:
        for seed in seed_list:
            A = gen_cond_matrix(CondSpec(m, n, kappa=float(kappa), seed=seed))
            for name, fn in algos.items():
                try:
                    Q, R = fn(A)
                    orth, res = _measures(A, Q, R)
                    ok = np.isfinite(orth) and np.isfinite(res)
                    rep.rows.append((name, float(kappa), seed, orth, res, "ok" if ok else "failed"))
                except (CholeskyFailure, DimensionError, RuntimeError):
                    rep.rows.append((name, float(kappa), seed, float("nan"), float("nan"), "failed"))
    return rep
