"""Per-GPU R-only TSQR time at the shard sizes of C3 on 1, 2, 4 and 8 GPUs (leaves of
8192 x 128), with and without CAQR_TUNE_FUSE.  One GPU; the cross-GPU tree is not included."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

for P in (2048, 1024, 512, 256):
    A = torch.randn(P * 8192, 128, dtype=torch.float64, device="cuda")
    for fuse in (148, 0):
        _lib.tune(_lib.TUNE_FUSE, fuse)
        for _ in range(3):
            factor_device(A, P)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            factor_device(A, P)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        fl = 2 * P * 8192 * 128 * 128 - 2 / 3 * 128 ** 3
        print(f"P={P} fuse={fuse}: {ms:.3f} ms  {fl / ms / 1e9:.2f} TF/s", flush=True)
    del A
_lib.reset_tuning()
