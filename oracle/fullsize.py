"""Full-size inputs of the five BASELINE configs, bit-for-bit (test oracle only).

Each config's matrix is drawn with the reference's own generators
(``rng_for`` = Philox(seed), core.py:31-33; ``gen_cond_matrix``,
core.py:165-177) exactly as SURVEY.md section 8(d) specifies, in row chunks:
numpy's Generator draws a C-ordered array element by element from one
stream, so consecutive chunk draws are bitwise-identical to one draw of the
whole matrix.  A SHA-256 over the C-order bytes identifies the input; the
fixtures in ``tests/golden/fullsize_*.npz`` (``oracle/make_fullsize.py``)
record it and the GPU tests check it before comparing results.

C2 goes through LAPACK (QR of seeded Gaussians), whose bits depend on the
OpenBLAS kernel family and thread count.  It is generated in a subprocess
pinned to ``OPENBLAS_CORETYPE=Haswell`` and one thread, which any AVX2 x86
host reproduces.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# (m, n, leaf_rows, distribution) per config; SURVEY.md section 8 table
CONFIGS = {
    "c1": (65536, 32, 8192, "normal"),
    "c2": (1 << 20, 64, 4096, "cond1e12"),
    "c3": (1 << 24, 128, 8192, "normal"),
    "c4": (1 << 27, 8, 16384, "uniform"),
    "c5": (16384, 16384, 2048, "normal"),
}
# rows per generation chunk (~0.5-1 GiB), the unit of the parallel regeneration
CHUNK_ROWS = {"c1": 65536, "c2": 1 << 20, "c3": 1 << 20, "c4": 1 << 23, "c5": 1024}
PINNED_BLAS = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1"}


def _draw(rng, dist, rows, n):
    if dist == "normal":
        return rng.standard_normal((rows, n))
    return rng.uniform(-1.0, 1.0, (rows, n))


def chunks(config, seed=0, chunk_rows=None, states=None):
    """Yield (row0, block) of the config's input in C order, chunk by chunk.

    ``states`` (a list) receives the Philox state at every chunk start
    (``pack_state``), from which ``parallel_chunks`` regenerates the chunks
    independently.
    """
    from paper_0809_2407_b200 import core

    m, n, _, dist = CONFIGS[config]
    chunk_rows = chunk_rows or CHUNK_ROWS[config]
    if dist == "cond1e12":
        A = cond_input(seed)
        for r in range(0, m, chunk_rows):
            yield r, A[r:r + chunk_rows]
        return
    rng = core.rng_for(seed)
    for r in range(0, m, chunk_rows):
        if states is not None:
            states.append(pack_state(rng.bit_generator.state))
        yield r, _draw(rng, dist, min(chunk_rows, m - r), n)


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


def parallel_chunks(config, states, sink, threads=8):
    """Regenerate every chunk from its recorded state on a thread pool (numpy
    releases the GIL while it fills) and call ``sink(row0, block)`` in chunk
    order.  Bitwise-identical to ``chunks`` (same stream, restored state)."""
    from concurrent.futures import ThreadPoolExecutor

    m, n, _, dist = CONFIGS[config]
    cr = CHUNK_ROWS[config]
    starts = list(range(0, m, cr))
    assert len(starts) == len(states), "state table does not match the chunking"

    def gen(i):
        bg = np.random.Philox(0)
        bg.state = unpack_state(states[i])
        return _draw(np.random.Generator(bg), dist, min(cr, m - starts[i]), n)

    with ThreadPoolExecutor(threads) as ex:
        futs = [ex.submit(gen, i) for i in range(min(threads, len(starts)))]
        for i, r0 in enumerate(starts):
            blk = futs[i].result()
            futs[i] = None
            if i + threads < len(starts):
                futs.append(ex.submit(gen, i + threads))
            sink(r0, blk)


def cond_input(seed=0):
    """C2's gen_cond_matrix(CondSpec(2**20, 64, 1e12, seed)) under the pinned BLAS."""
    m, n, _, _ = CONFIGS["c2"]
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "a.npy")
        code = (
            "import sys, numpy as np; sys.path.insert(0, %r);"
            "from paper_0809_2407_b200 import core;"
            "np.save(%r, core.gen_cond_matrix(core.CondSpec(%d, %d, kappa=1e12, seed=%d)))"
            % (ROOT, out, m, n, seed)
        )
        env = dict(os.environ, **PINNED_BLAS)
        subprocess.run([sys.executable, "-c", code], check=True, env=env)
        return np.load(out)


class Sha:
    def __init__(self):
        self.h = hashlib.sha256()

    def update(self, block):
        self.h.update(np.ascontiguousarray(block, dtype=np.float64).tobytes())

    def hexdigest(self):
        return self.h.hexdigest()


def power_norm2(matvec, rmatvec, n, iters=60, seed=0x5EED):
    """sigma_max by power iteration on A^T A (core.py:110-131's method)."""
    x = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = rmatvec(matvec(x))
        lam = float(np.linalg.norm(y))
        x = y / lam
    return float(np.sqrt(lam))
