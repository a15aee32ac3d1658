"""k_tree_factor_dmma vs k_tree_factor_w32 on one node (n = 8, P = 2): element differences of
node Y, tau, R, and per-reflector orthogonality |tau (1 + |y|^2) - 2|."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

for n in (8, 32):
    A = torch.from_numpy(np.random.default_rng(n).standard_normal((2 * 600, n))).cuda()
    out = []
    for tf in (1, 0):
        _lib.tune(_lib.TUNE_DMMA_TREE_FACTOR, tf)
        f = factor_device(A, 2, want_q=True)
        Y = f.node_Y[0].cpu().numpy()
        t = f.node_tau[0].cpu().numpy()
        out.append((Y, t, f.R.cpu().numpy()))
        # reflector j = [e_j; Y[:, j]]: orthogonal iff tau (1 + |y|^2) = 2 (or tau = 0)
        defect = [abs(t[j] * (1 + Y[:, j] @ Y[:, j]) - 2) if t[j] else 0.0 for j in range(n)]
        print(n, f"tree_factor={tf} max reflector defect {max(defect):.2e}",
              "Y lower max", np.abs(np.tril(Y, -1)).max())
    _lib.reset_tuning()
    print(n, "dY", np.abs(out[0][0] - out[1][0]).max(), "dtau", np.abs(out[0][1] - out[1][1]).max(),
          "dR", np.abs(out[0][2] - out[1][2]).max())
