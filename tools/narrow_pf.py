"""C4: k_leaf_narrow8 L2 prefetch distance sweep (graph replay, so the host does not bound it)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.tsqr import factor_device

m = 1 << 27
P = m // 16384
A = torch.rand(m, 8, dtype=torch.float64, device="cuda") * 2 - 1
for pf in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,0,1,2,4,6,8,12,3").split(",")]:
    _lib.tune(_lib.TUNE_NARROW_PF, pf)
    for _ in range(2):
        factor_device(A, P)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        factor_device(A, P, check=False)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"pf={pf}: {ms:.4f} ms {64 * m / ms / 1e6:.0f} GB/s", flush=True)
