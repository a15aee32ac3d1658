"""Randomised cross-check of the DMMA kernels against the rank-1 / reflector
rings on many shapes (n in (64,128], ragged leaves, narrow and wide applies)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import apply_q_device, factor_device

EPS = np.finfo(np.float64).eps
rng = np.random.default_rng(1234)
worst = 0.0
for it in range(40):
    n = int(rng.integers(65, 129))
    P = int(rng.integers(1, 9))
    m = P * int(rng.integers(max(n, 300), 3000)) + int(rng.integers(0, 50))
    k = int(rng.choice([int(rng.integers(1, 200)), int(rng.integers(2000, 6000))]))
    A = torch.from_numpy(rng.standard_normal((m, n))).cuda()
    C = torch.from_numpy(rng.standard_normal((m, k))).cuda()
    f = factor_device(A, P, want_q=True)
    R1 = factor_device(A, P).R
    Qd = apply_q_device(f, C, transpose=True)
    _lib.tune(_lib.TUNE_DMMA, 0)
    _lib.tune(_lib.TUNE_DMMA_APPLY, 0)
    f0 = factor_device(A, P, want_q=True)
    R0 = factor_device(A, P).R
    Qr = apply_q_device(f0, C, transpose=True)
    _lib.tune(_lib.TUNE_DMMA, 1)
    _lib.tune(_lib.TUNE_DMMA_APPLY, 1)
    sgn = lambda R: R * torch.sign(torch.diagonal(R)).unsqueeze(1)
    dR = (sgn(R1) - sgn(R0)).abs().max().item() / torch.linalg.norm(A, 2).item()
    dQ = (torch.linalg.norm(Qd - Qr) / torch.linalg.norm(C)).item()
    dY = (f.R - f0.R).abs().max().item() / torch.linalg.norm(A, 2).item()
    worst = max(worst, dR / EPS, dQ / EPS, dY / EPS)
    print(f"m={m:6d} n={n:3d} P={P} k={k:5d}: R-only {dR / EPS:6.1f} eps, Q-path R {dY / EPS:6.1f} eps, Q^T C {dQ / EPS:7.1f} eps")
print(f"worst {worst:.1f} eps")
assert worst < 1000
