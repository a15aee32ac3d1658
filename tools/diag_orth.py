"""Orthogonality of explicit Q at small n under the DMMA tree-factor / leaf-Q switches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

for n in (8, 17, 32, 64, 100, 128):
    m, P = 8 * 600 + 3, 8
    A = np.random.Generator(np.random.Philox(31 * n)).standard_normal((m, n))
    At = torch.from_numpy(A).cuda()
    for tf in ((1, 0) if n <= 64 else (0,)):
        for dq in (1,):
            for tr in (1,):
                _lib.tune(_lib.TUNE_DMMA_TREE_FACTOR, tf)
                _lib.tune(_lib.TUNE_DMMA_Q, dq)
                _lib.tune(_lib.TUNE_DMMA_TREE, tr)
                f = factor_device(At, P, want_q=True)
                Q = explicit_q_device(f).cpu().numpy()
                print(n, f"tree_factor={tf} leaf_q={dq} tree_apply={tr}",
                      f"orth/(n eps)={oracle.orthogonality(Q) / (n * oracle.EPS):.2f}",
                      f"resid/(n eps)={oracle.residual(A, Q, f.R.cpu().numpy()) / (n * oracle.EPS):.2f}")
    _lib.reset_tuning()
