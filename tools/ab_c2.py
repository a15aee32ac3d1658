"""A/B of the C2 step (1048576 x 64, leaves of 4096, R + explicit Q) under tuning settings:
(CAQR_TUNE_DMMA, CAQR_TUNE_CHAIN_HT_64, CAQR_TUNE_DMMA_Q), interleaved rounds, CUDA-event timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

m, n, P = 1048576, 64, 256
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
settings = [(2, 16, 1, 1, 1), (2, 16, 1, 1, 0)]
res = {s: [] for s in settings}


def step():
    f = factor_device(A, P, want_q=True, check=False)
    return explicit_q_device(f)


for rnd in range(5):
    for s in settings:
        _lib.tune(_lib.TUNE_DMMA, s[0])
        _lib.tune(_lib.TUNE_CHAIN_HT[64], s[1])
        _lib.tune(_lib.TUNE_DMMA_Q, s[2])
        _lib.tune(_lib.TUNE_DMMA_TREE, s[3])
        _lib.tune(_lib.TUNE_DMMA_TREE_FACTOR, s[4])
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            step()
        e1.record()
        torch.cuda.synchronize()
        res[s].append(e0.elapsed_time(e1) / 10)
for s in settings:
    v = sorted(res[s])
    print(f"dmma={s[0]} ht64={s[1]} dmma_q={s[2]} dmma_tree={s[3]} tree_factor={s[4]}: median {v[len(v) // 2]:.3f} ms  min {v[0]:.3f}")
_lib.reset_tuning()
