import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import _leaf_apply, factor_device
m, n, k = 16384, 128, 16256
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
C = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
for leaf in (2048, 512):
    _lib.tune(_lib.TUNE_CHAIN_HT[128], 64)
    f = factor_device(A, m // leaf, want_q=True)
    for _ in range(2):
        _leaf_apply(f, C, transpose=True)
torch.cuda.synchronize()
