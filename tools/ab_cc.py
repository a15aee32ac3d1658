"""A/B of the C3 leaf factorisation: split-role ring (CAQR_TUNE_CC=2) vs the DMMA
warp ring (0), on one wave of leaves and on the full C3 step, with R compared
between the two (sign-normalised) and against LAPACK on the CPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

EPS = float(np.finfo(np.float64).eps)


def sn(R):
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1
    return d[:, None] * R


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (m, n, P) in [(148 * 8192, 128, 148), (1 << 24, 128, 2048), (148 * 8192, 96, 148), (300 * 1000 + 77, 72, 300)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    out = {}
    for cc in (4, 3, 0):
        _lib.tune(_lib.TUNE_CC, cc)
        ms = timed(lambda: factor_device(A, P, check=False))
        out[cc] = (ms, factor_device(A, P).R_out().clone())
    flops = 2 * m * n * n - 2 * n ** 3 / 3
    nrm = float(torch.linalg.matrix_norm(out[0][1], 2))
    line = f"m={m} n={n} P={P}:"
    for cc, name in ((4, "tmem16"), (3, "tmem12"), (0, "ring")):
        d = float(torch.max(torch.abs(sn(out[cc][1]) - sn(out[0][1])))) / nrm / EPS
        line += f"  {name} {out[cc][0]:.3f} ms ({flops / out[cc][0] / 1e9:.2f} TF/s, dR {d:.2f})"
    print(line, flush=True)
    if m <= 1 << 21:
        Rl = torch.as_tensor(np.linalg.qr(A.cpu().numpy(), mode="r"), device="cuda")
        d2 = float(torch.max(torch.abs(sn(out[4][1]) - sn(Rl)))) / float(torch.linalg.matrix_norm(Rl, 2)) / EPS
        print(f"   |R_tmem16 - R_lapack| = {d2:.2f} eps*|A|_2", flush=True)
_lib.reset_tuning()
