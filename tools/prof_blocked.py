"""Blocked tall-tile leaf (CAQR_TUNE_BLOCKED) vs the warp ring: parity and timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

for (m, n, P) in [(4096, 128, 2), (20000, 100, 4), (3000, 70, 1), (9000, 128, 3)]:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    _lib.tune(_lib.TUNE_BLOCKED, 1)
    Rb = factor_device(A, P).R.cpu().numpy()
    _lib.tune(_lib.TUNE_BLOCKED, 0)
    Rr = factor_device(A, P).R.cpu().numpy()
    Rl = np.linalg.qr(A.cpu().numpy(), mode="r")
    sc = np.linalg.norm(A.cpu().numpy(), 2)
    print(f"{m}x{n} P={P}: blocked vs LAPACK {oracle.r_diff(Rb, Rl, sc) / oracle.EPS:.1f} eps, "
          f"ring vs LAPACK {oracle.r_diff(Rr, Rl, sc) / oracle.EPS:.1f} eps")
m, n, P = 148 * 8192, 128, 148
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
for mode in (0, 1, 0, 1):
    _lib.tune(_lib.TUNE_BLOCKED, mode)
    for _ in range(2):
        factor_device(A, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    factor_device(A, P, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{'blocked' if mode else 'ring   '}: {ms:.3f} ms, {(2 * m * n * n - 2 * n ** 3 / 3) / ms / 1e9:.2f} TFLOP/s")
_lib.tune(_lib.TUNE_BLOCKED, 0)
