"""C4 kernel timing modes: sizes, back-to-back vs isolated launches, row order of leaves."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

def t_loop(A, P, reps=5):
    for _ in range(2):
        factor_device(A, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        factor_device(A, P, check=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for lg in (24, 25, 26, 27):
    m = 1 << lg
    A = torch.rand(m, 8, dtype=torch.float64, device="cuda") * 2 - 1
    for leaf in (16384, 65536, 4096):
        ms = t_loop(A, m // leaf)
        print(f"m=2^{lg} leaf={leaf}: {ms:.4f} ms {64 * m / ms / 1e6:.0f} GB/s", flush=True)
    if lg == 27:
        P = m // 16384
        ts = []
        for i in range(8):
            torch.cuda.synchronize(); time.sleep(0.05)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); factor_device(A, P, check=False); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print("isolated:", " ".join(f"{t:.3f}" for t in ts))
        # plain read bandwidth of the same buffer
        for _ in range(2): s = A.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): s = A.sum()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"torch sum: {ms:.4f} ms {64 * m / ms / 1e6:.0f} GB/s")
    del A
