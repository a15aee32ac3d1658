"""Time caqr_factor (C5 shape by default) with and without lookahead / panel splitting."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200.caqr import caqr_factor

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--leaf", type=int, default=2048)
ap.add_argument("--variants", default="0:1,1:1,1:2,1:4")
a = ap.parse_args()
A = torch.randn(a.n, a.n, dtype=torch.float64, device="cuda")
fl = 4.0 / 3.0 * a.n ** 3
for var in a.variants.split(","):
    la, pc = (int(x) for x in var.split(":"))
    caqr_factor(A, b=128, leaf_rows=a.leaf, lookahead=bool(la), panel_chains=pc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    caqr_factor(A, b=128, leaf_rows=a.leaf, lookahead=bool(la), panel_chains=pc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"lookahead={la} panel_chains={pc}: {ms:.1f} ms, {fl / ms / 1e9:.2f} TFLOP/s")
