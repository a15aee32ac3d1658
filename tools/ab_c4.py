"""A/B of the C4 step (134217728 x 8 U(-1,1), leaves of 16384, R only): the
K = 8 narrow kernel (CAQR_TUNE_NARROW = 3) vs the cp.async K = 4 kernel (2),
interleaved rounds, CUDA events; R compared between them and with LAPACK on a
slice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

EPS = float(np.finfo(np.float64).eps)
m, n, P = 1 << 27, 8, 8192
g = torch.Generator(device="cuda").manual_seed(4)
A = torch.rand(m, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
res = {2: [], 3: []}
Rs = {}
for rnd in range(5):
    for v in (3, 2):
        _lib.tune(_lib.TUNE_NARROW, v)
        for _ in range(2):
            factor_device(A, P, check=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            factor_device(A, P, check=False)
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / 10)
        Rs[v] = factor_device(A, P).R_out()


def sn(R):
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1
    return d[:, None] * R


for v in (3, 2):
    t = sorted(res[v])[2]
    print(f"narrow={v}: median {t:.3f} ms  {8 * m * n / t / 1e6:.0f} GB/s  "
          f"({8 * m * n / t / 1e6 / 6538.9 * 100:.1f}% of 6538.9)")
nrm = float(torch.linalg.matrix_norm(Rs[2], 2))
print("max |sn(R3) - sn(R2)| =", float(torch.max(torch.abs(sn(Rs[3]) - sn(Rs[2])))) / nrm / EPS, "eps*|A|")
for (mm, PP) in [(1 << 20, 64), (300000 + 7, 9), (5000, 1)]:
    B = A[:mm]
    for v in (3, 2):
        _lib.tune(_lib.TUNE_NARROW, v)
        R = factor_device(B, PP).R_out()
        Rl = torch.as_tensor(np.linalg.qr(B.cpu().numpy(), mode="r"), device="cuda")
        print(f"  m={mm} P={PP} narrow={v}: |sn(R) - sn(R_lapack)| = "
              f"{float(torch.max(torch.abs(sn(R) - sn(Rl)))) / float(torch.linalg.matrix_norm(Rl, 2)) / EPS:.2f} eps*|A|")
_lib.reset_tuning()
