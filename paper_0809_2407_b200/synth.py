"""The five BASELINE configs' inputs, bit for bit the reference's.

Every matrix is drawn with the reference's own generators: ``rng_for(seed)``
(Philox, core.py:31-33) C-order draws for C1 / C3 / C4 / C5 and
``gen_cond_matrix(CondSpec(2**20, 64, 1e12, seed))`` (core.py:165-177) for C2.
numpy's Generator fills an array from one sequential stream, so a row range
is regenerated independently from the Philox state at the start of its chunk:
``data/synth_states.npz`` holds those states (recorded once by a sequential
pass, oracle/make_fullsize.py ``states``), and chunks are drawn on a thread
pool (numpy releases the GIL while it fills) and copied to the device.  The
bench uses this to time the exact inputs the reference would see, shard by
shard under torchrun, and to check the timed R against the reference's.

C2 goes through LAPACK (QR of seeded Gaussians), whose bits depend on the
OpenBLAS kernel family and thread count; it is generated in a subprocess
pinned to ``OPENBLAS_CORETYPE=Haswell`` and one thread.
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

# (m, n, leaf_rows, distribution) per config
CONFIGS = {
    "c1": (65536, 32, 8192, "normal"),
    "c2": (1 << 20, 64, 4096, "cond1e12"),
    "c3": (1 << 24, 128, 8192, "normal"),
    "c4": (1 << 27, 8, 16384, "uniform"),
    "c5": (16384, 16384, 2048, "normal"),
}
# rows per generation chunk (~0.5-1 GiB), the unit of parallel regeneration
CHUNK_ROWS = {"c1": 65536, "c2": 1 << 20, "c3": 1 << 20, "c4": 1 << 23, "c5": 1024}
PINNED_BLAS = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1"}


def draw(rng, dist, rows, n):
    if dist == "normal":
        return rng.standard_normal((rows, n))
    return rng.uniform(-1.0, 1.0, (rows, n))


def pack_state(st):
    """Philox state dict -> 13 uint64 (counter 4, key 2, buffer 4, pos, has_u32, u32)."""
    s = st["state"]
    return np.concatenate([s["counter"], s["key"], st["buffer"],
                           np.array([st["buffer_pos"], st["has_uint32"], st["uinteger"]],
                                    dtype=np.uint64)]).astype(np.uint64)


def unpack_state(a):
    a = np.asarray(a, dtype=np.uint64)
    return {"bit_generator": "Philox",
            "state": {"counter": a[0:4].copy(), "key": a[4:6].copy()},
            "buffer": a[6:10].copy(), "buffer_pos": int(a[10]), "has_uint32": int(a[11]),
            "uinteger": int(a[12])}


def state_table(config):
    return np.load(os.path.join(HERE, "data", "synth_states.npz"))[f"{config}_states"]


def cond_input(seed=0):
    """C2's gen_cond_matrix(CondSpec(2**20, 64, 1e12, seed)) under the pinned BLAS."""
    m, n, _, _ = CONFIGS["c2"]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "a.npy")
        code = ("import sys, numpy as np; sys.path.insert(0, %r);"
                "from paper_0809_2407_b200 import core;"
                "np.save(%r, core.gen_cond_matrix(core.CondSpec(%d, %d, kappa=1e12, seed=%d)))"
                % (ROOT, out, m, n, seed))
        subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, **PINNED_BLAS))
        return np.load(out)


def chunks(config, lo=0, hi=None, sink=None, threads=8):
    """Rows [lo, hi) of the config's seed-0 input, chunk by chunk, in order:
    ``sink(row0, block)`` per generated block (blocks are clipped to [lo, hi)).
    C3 / C4 / C5 regenerate only the chunks that overlap the range, from the
    recorded Philox states, on ``threads`` threads; C1 / C2 draw sequentially."""
    from .core import rng_for

    m, n, _, dist = CONFIGS[config]
    hi = m if hi is None else hi
    if config == "c2":
        A = cond_input(0)
        sink(lo, A[lo:hi])
        return
    if config == "c1":
        A = draw(rng_for(0), dist, m, n)
        sink(lo, A[lo:hi])
        return
    cr = CHUNK_ROWS[config]
    states = state_table(config)
    idx = list(range(lo // cr, (hi - 1) // cr + 1))

    def gen(i):
        bg = np.random.Philox(0)
        bg.state = unpack_state(states[i])
        blk = draw(np.random.Generator(bg), dist, min(cr, m - i * cr), n)
        a, b = max(lo, i * cr), min(hi, (i + 1) * cr)
        return a, blk[a - i * cr:b - i * cr]

    with ThreadPoolExecutor(threads) as ex:
        futs = [ex.submit(gen, i) for i in idx[:threads]]
        for j in range(len(idx)):
            r0, blk = futs[j].result()
            futs[j] = None
            if j + threads < len(idx):
                futs.append(ex.submit(gen, idx[j + threads]))
            sink(r0, blk)


def device_input(config, device, lo=0, hi=None):
    """Rows [lo, hi) of the config's input as a CUDA tensor (pinned staging)."""
    import torch

    m, n, _, _ = CONFIGS[config]
    hi = m if hi is None else hi
    A = torch.empty((hi - lo, n), dtype=torch.float64, device=device)
    pin = {"t": torch.empty(0, dtype=torch.float64)}

    def sink(r0, blk):
        t = torch.from_numpy(np.ascontiguousarray(blk))
        if pin["t"].numel() < t.numel():
            pin["t"] = torch.empty(t.numel(), dtype=torch.float64).pin_memory()
        torch.cuda.current_stream(device).synchronize()
        buf = pin["t"][:t.numel()]
        buf.copy_(t.reshape(-1))
        A[r0 - lo:r0 - lo + blk.shape[0]].copy_(buf.view(blk.shape), non_blocking=True)

    chunks(config, lo, hi, sink)
    torch.cuda.current_stream(device).synchronize()
    return A
