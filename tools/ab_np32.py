"""A/B of Q^T C at n = 32 (2^20 x 32, 128 leaves, k = 32 / 256): reflector ring
(CAQR_TUNE_DMMA_APPLY = 0) vs k_leaf_q_dmma<32> (= 4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import apply_q_device, factor_device

A = torch.randn(1 << 20, 32, dtype=torch.float64, device="cuda")
f = factor_device(A, 128, want_q=True, check=False)
for k in (32, 256):
    C = torch.randn(1 << 20, k, dtype=torch.float64, device="cuda")
    for av in (0, 4, 0, 4):
        _lib.tune(_lib.TUNE_DMMA_APPLY, av)
        for _ in range(3):
            apply_q_device(f, C, True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            apply_q_device(f, C, True)
        e1.record()
        torch.cuda.synchronize()
        print(f"Q^T C 2^20x32 k={k} dmma_apply={av}: {e0.elapsed_time(e1) / 10:.3f} ms")
_lib.reset_tuning()
