"""Per-launch time of one tree level (stacked-triangle combine with node factors
kept, and its Q^T apply) for n = 32 / 64 / 128 and 1 / 8 / 128 events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib


def ptr(t):
    return t.data_ptr()


lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
for n in (32, 64, 128):
    for nev in (1, 8, 128):
        P = 2 * nev
        Rs = torch.triu(torch.randn(P, n, n, dtype=torch.float64, device="cuda"))
        ev = torch.tensor([[2 * e, 2 * e + 1, e] for e in range(nev)], dtype=torch.int32,
                          device="cuda")
        Y = torch.empty(nev, n, n, dtype=torch.float64, device="cuda")
        tau = torch.empty(nev, n, dtype=torch.float64, device="cuda")
        C = torch.randn(P * n, n, dtype=torch.float64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        for it in range(2):
            R0 = Rs.clone()
            e0.record()
            for _ in range(reps):
                _lib.check(lib.tsqr_f64_tree_factor_level(ptr(R0), n, ptr(ev), nev, ptr(Y), ptr(tau),
                                                          st), "factor")
            e1.record()
            torch.cuda.synchronize()
        tf = e0.elapsed_time(e1) / reps * 1e3
        for it in range(2):
            e0.record()
            for _ in range(reps):
                _lib.check(lib.tsqr_f64_tree_apply_level(ptr(Y), ptr(tau), n, ptr(ev), nev, ptr(C), n,
                                                         n, n, 1, 0, st), "apply")
            e1.record()
            torch.cuda.synchronize()
        ta = e0.elapsed_time(e1) / reps * 1e3
        print(f"n={n:3d} events={nev:4d}: factor {tf:7.1f} us  apply {ta:7.1f} us")
