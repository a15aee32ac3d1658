"""Pinned host -> device copy bandwidth: one stream vs two / four streams (1 GiB chunks)."""
import torch

n = 1 << 27  # 1 GiB of doubles
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(8):
            s = streams[i % ns]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i % 4].copy_(h[i % 4], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"{ns} stream(s): {8 * 8 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
