"""A/B of the C5 step (CAQR 16384^2, b = 128, leaf 2048) over caqr_factor
settings (apply_waves, panel_chains), CUDA events, R checked against the
first setting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200.caqr import caqr_factor

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
settings = [(0.0, 4), (1.0, 4), (2.0, 4), (4.0, 4)]
Rs = {}
for s in settings:
    for _ in range(2):
        caqr_factor(A, b=128, leaf_rows=2048, apply_waves=s[0], panel_chains=s[1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        res = caqr_factor(A, b=128, leaf_rows=2048, apply_waves=s[0], panel_chains=s[1])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    R = res.R
    d = torch.sign(torch.diagonal(R)); d[d == 0] = 1
    Rs[s] = d[:, None] * R
    dr = float(torch.max(torch.abs(Rs[s] - Rs[settings[0]]))) / float(torch.max(torch.abs(Rs[settings[0]])))
    F = 2 * n ** 3 - 2 * n ** 3 / 3
    print(f"apply_waves={s[0]} panel_chains={s[1]}: {ms:.1f} ms  {F / ms / 1e9:.0f} GF/s "
          f"({F / ms / 1e9 / 37225 * 100:.1f}% of FP64 peak)  rel dR {dr:.2e}", flush=True)
