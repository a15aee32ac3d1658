import time, torch, sys
sys.path.insert(0, '.')
from paper_0809_2407_b200.caqr import caqr_factor
n = 16384
A = torch.randn(n, n, dtype=torch.float64, device='cuda')
Ah = torch.empty(A.shape, dtype=torch.float64, pin_memory=True); Ah.copy_(A)
for la in (True, False):
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = caqr_factor(Ah, b=128, leaf_rows=2048, lookahead=la)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        R = res.R
        t2 = time.perf_counter()
        del res, R
        print(f"lookahead={la} it={it}: factor(host in) {1e3*(t1-t0):.0f} ms, R to host {1e3*(t2-t1):.0f} ms", flush=True)
