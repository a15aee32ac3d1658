"""Small driver for ncu: one TSQR factor_device call per config (n, leaves, leaf rows)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200.tsqr import factor_device, explicit_q_device

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--leaves", type=int, default=148)
ap.add_argument("--leaf-rows", type=int, default=8192)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--q", default="none")
ap.add_argument("--ht", type=int, default=0)
ap.add_argument("--tune", action="append", default=[], help="KEY=VALUE (caqr_tune)")
a = ap.parse_args()
from paper_0809_2407_b200 import _lib
np_ = 32 if a.n <= 32 else (64 if a.n <= 64 else 128)
for kv in a.tune:
    k, v = kv.split("=")
    _lib.tune(int(k), int(v))
if a.ht:
    _lib.tune(_lib.TUNE_CHAIN_HT[np_], a.ht)
A = torch.randn(a.leaves * a.leaf_rows, a.n, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    f = factor_device(A, a.leaves, want_q=a.q != "none")
    if a.q == "explicit":
        explicit_q_device(f)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f = factor_device(A, a.leaves, want_q=a.q != "none")
if a.q == "explicit":
    explicit_q_device(f)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
m, n = A.shape
print(f"n={n} leaves={a.leaves} rows={a.leaf_rows}: {ms:.3f} ms, {(2*m*n*n - 2*n**3/3)/ms/1e9:.2f} TFLOP/s ht={_lib.geometry(a.n)[2]}")
