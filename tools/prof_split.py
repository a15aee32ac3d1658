"""Time factor_device (R only, or R + explicit Q) for a shape at several chain splits."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200.tsqr import _leaves_for, explicit_q_device, factor_device

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1 << 21)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--leaf", type=int, default=8192)
ap.add_argument("--ks", default="1,2,4,8")
ap.add_argument("--q", action="store_true")
a = ap.parse_args()
A = torch.randn(a.m, a.n, dtype=torch.float64, device="cuda")
P0 = _leaves_for(a.m, a.n, a.leaf)
for k in [int(x) for x in a.ks.split(",")]:
    P = P0 * k
    def run():
        f = factor_device(A, P, want_q=a.q)
        if a.q:
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
    print(f"m={a.m} n={a.n} P={P0}x{k}: {e0.elapsed_time(e1) / 3:.3f} ms")
