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
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_0809_2407_b200.synth import (  # noqa: E402,F401  (the product's generator)
    CHUNK_ROWS,
    CONFIGS,
    PINNED_BLAS,
    cond_input,
    draw as _draw,
    pack_state,
    unpack_state,
)


def chunks(config, seed=0, chunk_rows=None, states=None):
    """Yield (row0, block) of the config's input in C order by a SEQUENTIAL
    pass of the reference generator (no state table needed); ``states`` (a
    list) receives the Philox state at every chunk start -- the table
    paper_0809_2407_b200/synth.py regenerates chunks from."""
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
