"""One CAQR panel-0 style factor + trailing update with the kept panel T (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0809_2407_b200 import _lib
m, n, k, P = 16384, 128, 16256, 8
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
C = torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g)
_, h0, ht = _lib.geometry(n)
tiles = 1 + -(-(m // P - h0) // ht)
tau = torch.zeros(P, tiles, n, dtype=torch.float64, device="cuda")
Rs = torch.empty(P, n, n, dtype=torch.float64, device="cuda")
T = torch.empty(P * tiles * 1024, dtype=torch.float64, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
Y = A.clone()
_lib.check(lib.tsqr_f64_leaf_factor_t(Y.data_ptr(), n, m, n, P, Y.data_ptr(), n, tau.data_ptr(), tiles * n,
                                      Rs.data_ptr(), flag.data_ptr(), T.data_ptr(), st), "factor_t")
import os
for _ in range(3):
    _lib.check(lib.tsqr_f64_leaf_apply_t(Y.data_ptr(), n, tau.data_ptr(), tiles * n, m, n, P, C.data_ptr(), k, k,
                                         T.data_ptr(), st), "apply_t")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.check(lib.tsqr_f64_leaf_apply_t(Y.data_ptr(), n, tau.data_ptr(), tiles * n, m, n, P, C.data_ptr(), k, k,
                                     T.data_ptr(), st), "apply_t")
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"apply_t {ms:.3f} ms  {4.0 * m * n * k / ms / 1e9:.2f} TF/s")
