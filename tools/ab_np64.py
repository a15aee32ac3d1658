"""A/B of the n <= 64 / explicit-Q paths under tuning settings (interleaved rounds, CUDA events):
R only at n = 64 (chain vs DMMA ring), Q^T C at n = 64 (chain tile 24 vs 16), explicit Q at
n = 128 (reflector ring vs DMMA Q)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device, factor_device

D, H, Q = _lib.TUNE_DMMA, _lib.TUNE_CHAIN_HT[64], _lib.TUNE_DMMA_Q


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


A64 = torch.randn(1 << 21, 64, dtype=torch.float64, device="cuda")
A128 = torch.randn(1 << 20, 128, dtype=torch.float64, device="cuda")
C64 = torch.randn(1 << 21, 64, dtype=torch.float64, device="cuda")
cases = {
    "R only 2^21x64 P=512, dmma 1": ({D: 1}, lambda: factor_device(A64, 512, check=False)),
    "R only 2^21x64 P=512, dmma 2": ({D: 2}, lambda: factor_device(A64, 512, check=False)),
    "R only 2^21x64 P=256, dmma 1": ({D: 1}, lambda: factor_device(A64, 256, check=False)),
    "R only 2^21x64 P=256, dmma 2": ({D: 2}, lambda: factor_device(A64, 256, check=False)),
}
res = {k: [] for k in cases}
for rnd in range(3):
    for k, (tn, fn) in cases.items():
        for key, v in tn.items():
            _lib.tune(key, v)
        res[k].append(timeit(fn))
        _lib.tune(D, 1)
for k in cases:
    print(f"{k}: {min(res[k]):.3f} ms")

for ht, av in ((24, 0), (16, 0), (16, 1), (16, 2), (16, 3)):
    _lib.tune(H, ht)
    _lib.tune(_lib.TUNE_DMMA_APPLY, av)
    f = factor_device(A64, 512, want_q=True, check=False)
    print(f"Q^T C 2^21x64 (k=64) ht64={ht} dmma_apply={av}: "
          f"{timeit(lambda: apply_q_device(f, C64, True)):.3f} ms")
_lib.reset_tuning()
f = factor_device(A128, 128, want_q=True, check=False)
for qv in (0, 1):
    _lib.tune(Q, qv)
    print(f"explicit Q 2^20x128 P=128 dmma_q={qv}: {timeit(lambda: explicit_q_device(f)):.3f} ms")
_lib.tune(Q, 1)
