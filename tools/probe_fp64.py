"""FP64 pipe microbenchmark on the GPU: DFMA chains vs DMMA m8n8k4 (libcaqr_sm100)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_0809_2407_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda")
scratch = torch.zeros(4, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream().cuda_stream
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = {"sms": sms}
for mode, name, fl_per_it in ((0, "dfma", 16 * 2 * 256), (1, "dmma_m8n8k4", 8 * 2 * 256 * 8)):
    for blocks_per_sm in (2, 4, 8):
        blocks = sms * blocks_per_sm
        iters = 20000
        lib.caqr_f64_peak_probe(scratch.data_ptr(), mode, 100, blocks, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.caqr_f64_peak_probe(scratch.data_ptr(), mode, iters, blocks, st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        # dfma: per thread per iter 16 FMA (2 flop); dmma: per warp per iter 8 mma x 256 FMA
        if mode == 0:
            fl = blocks * 256 * iters * 16 * 2
        else:
            fl = blocks * 8 * iters * 8 * 256 * 2
        out[f"{name}_{blocks_per_sm}cta"] = fl / ms / 1e9
print(json.dumps(out))
