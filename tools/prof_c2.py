"""C2 shape (R + explicit Q, n = 64) at chain tile heights 32 / 24 / 16."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

m, n, P = 1 << 20, 64, 256
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
for ht in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,24,16,32,24").split(",")]:
    _lib.tune(_lib.TUNE_CHAIN_HT[64], ht)
    for q in (False, True):
        def run():
            f = factor_device(A, P, want_q=True)
            if q:
                explicit_q_device(f)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"ht={ht} {'factor+Q' if q else 'factor  '}: {e0.elapsed_time(e1) / 3:.3f} ms")
