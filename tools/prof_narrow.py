"""C4-shaped R-only TSQR (n = 8) with the narrow kernel variants (CAQR_TUNE_NARROW 1 / 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
P = m // 16384
A = torch.rand(m, 8, dtype=torch.float64, device="cuda") * 2 - 1
for mode in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,2,3").split(",")]:
    _lib.tune(_lib.TUNE_NARROW, mode)
    for _ in range(2):
        factor_device(A, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        factor_device(A, P, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"narrow={mode} m={m}: {ms:.3f} ms, {8 * m * 8 / ms / 1e6:.0f} GB/s")
