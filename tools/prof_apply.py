"""One CAQR-like leaf-level trailing update (k_leaf_apply transpose) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200.tsqr import _leaf_apply, factor_device

m, n, P, k = 16384, 128, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 16384 - 128
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
f = factor_device(A, P, want_q=True)
C = torch.randn(m, k, dtype=torch.float64, device="cuda")
for _rep in range(1):
    for _ in range(2):
        _leaf_apply(f, C, transpose=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _leaf_apply(f, C, transpose=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"leaf apply Q^T: {ms:.3f} ms, {4.0 * m * n * k / ms / 1e9:.2f} TFLOP/s")
