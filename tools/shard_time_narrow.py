"""Per-GPU R-only TSQR time at the shard sizes of C4 on 1, 2, 4 and 8 GPUs (leaves of 16384 x 8),
through tsqr.split_leaves(narrow=True) and without it.  Graph replay; one GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0809_2407_b200.tsqr import factor_device, split_leaves

for P in (8192, 4096, 2048, 1024, 64):
    m = P * 16384
    A = torch.rand(m, 8, dtype=torch.float64, device="cuda") * 2 - 1
    for k in (split_leaves(m, 8, P, narrow=True), 1):
        for _ in range(2):
            factor_device(A, P * k)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            factor_device(A, P * k, check=False)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"P={P} chains/leaf={k}: {ms:.4f} ms  {64 * m / ms / 1e6:.0f} GB/s", flush=True)
    del A
