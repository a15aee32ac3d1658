"""A/B of the CAQR panel kernels at C5's first-panel shape: 16-row chain tiles
(k_leaf_dmma ring + k_leaf_apply_dmma) vs tall 64-row tiles (k_leaf_tt<64,1,true> +
k_tall_apply): leaf factor with kept Q, the leaf-level trailing update Q^T C on
16256 columns and on the 128 look-ahead columns."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import _leaf_apply, factor_device


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


m, n = 16384, 128
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
for leaf in (512, 2048):
    P = m // leaf
    for ht in (16, 64):
        _lib.tune(_lib.TUNE_CHAIN_HT[128], ht)
        f = factor_device(A, P, want_q=True)
        tf = timed(lambda: factor_device(A, P, want_q=True, check=False))
        line = f"leaf {leaf:5d} ht {ht:2d}: factor (leaves + tree) {tf:7.3f} ms"
        for k in (16256, 4096, 128):
            C = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
            ta = timed(lambda: _leaf_apply(f, C, transpose=True))
            fl = 4.0 * m * n * k
            line += f" | Q^T C k={k}: {ta:7.3f} ms ({fl / ta / 1e9:5.2f} TF/s)"
        print(line, flush=True)
_lib.reset_tuning()
