"""Full-size parity fixtures for C2-C5 by running the READ-ONLY reference itself.

Run in the build container (where /root/reference exists), one config at a time:

    python oracle/make_fullsize.py c2|c3|c4|c5

For every config the input comes from ``oracle.fullsize.chunks`` (the
reference generators), hashed while it streams.

* TSQR configs (C2, C3, C4): the reference kernels composed as Algorithm 1
  (SPEC.md:295-302): ``qr_unblocked`` on every leaf of
  ``BlockRowLayout(m, n, P)`` (householder.py:128-145), then
  ``qr_stacked_triangles`` over ``ReductionTree(P, "binary").schedule()``
  (householder.py:263-294, trees.py:146-152).  Plus LAPACK's R of the whole
  matrix (streamed ``[R; chunk]`` QRs) as an independent check.
* C5: the reference's ``qr_blocked(A, nb=128)`` (householder.py:189-211, the
  Pr = Pc = 1 CAQR degenerate) and LAPACK ``dgeqrf``.  R is
  16384^2 (2 GiB), so the fixture keeps the sign-normalised diagonal, 8 full
  rows and sn(R) x for a seeded x; plus sigma_max by power iteration.

Nothing is copied from the reference: the script calls its public functions
and stores their outputs.  Fixtures: ``tests/golden/fullsize_<cfg>.npz``.
"""

from __future__ import annotations

import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import fullsize  # noqa: E402
from oracle.make_golden import load_reference  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
C5_ROWS = np.array([0, 1, 127, 128, 4095, 8191, 12288, 16383])
C5_X_SEED = 12345


def _init_worker():
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)


def _leaf_r(block):
    hh = load_reference()["householder"]
    return hh.qr_unblocked(block)[1]


def _sn(R):
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return d[:, None] * R


def tsqr_fixture(cfg):
    ref = load_reference()
    hh, trees, core = ref["householder"], ref["trees"], ref["core"]
    m, n, leaf, _ = fullsize.CONFIGS[cfg]
    P = m // leaf
    offs = core.BlockRowLayout(m, n, P).row_offsets()
    assert all(offs[i + 1] - offs[i] == leaf for i in range(P))
    sha = fullsize.Sha()
    Rlap = np.zeros((0, n))
    Rs = []
    t0 = time.time()
    with Pool(8, initializer=_init_worker) as pool:
        for r0, blk in fullsize.chunks(cfg):
            sha.update(blk)
            leaves = [blk[i:i + leaf] for i in range(0, blk.shape[0], leaf)]
            Rs.extend(pool.map(_leaf_r, leaves, chunksize=max(1, len(leaves) // 32)))
            Rlap = np.linalg.qr(np.vstack([Rlap, blk]), mode="r")
            print(f"{cfg}: rows {r0 + blk.shape[0]}/{m}  {time.time() - t0:.0f}s", flush=True)
    assert len(Rs) == P
    for ev in trees.ReductionTree(P=P, shape="binary").schedule():
        a, b = ev.participants
        Rs[a] = hh.qr_stacked_triangles([Rs[a], Rs[b]])[1]
    Rref = Rs[0]
    norm2 = float(np.linalg.svd(Rref, compute_uv=False)[0])
    d = float(np.max(np.abs(_sn(Rref) - _sn(Rlap))) / norm2)
    print(f"{cfg}: reference vs LAPACK R: {d / np.finfo(float).eps:.2f} eps*||A||_2", flush=True)
    np.savez_compressed(os.path.join(OUT, f"fullsize_{cfg}.npz"), sha256=sha.hexdigest(),
                        R_ref=Rref, R_lapack=Rlap, norm2=norm2, m=m, n=n, leaf_rows=leaf, P=P)


def c5_fixture():
    ref = load_reference()
    hh = ref["householder"]
    m, n, _, _ = fullsize.CONFIGS["c5"]
    sha = fullsize.Sha()
    A = np.empty((m, n))
    for r0, blk in fullsize.chunks("c5"):
        sha.update(blk)
        A[r0:r0 + blk.shape[0]] = blk
    x = np.random.Generator(np.random.Philox(C5_X_SEED)).standard_normal(n)
    out = {"sha256": sha.hexdigest(), "rows": C5_ROWS, "x_seed": C5_X_SEED, "m": m, "n": n}
    t0 = time.time()
    Rl = _sn(np.linalg.qr(A, mode="r"))
    print(f"c5: LAPACK {time.time() - t0:.0f}s", flush=True)
    out["lapack_diag"] = np.diag(Rl).copy()
    out["lapack_rows"] = Rl[C5_ROWS].copy()
    out["lapack_Rx"] = Rl @ x
    out["norm2"] = fullsize.power_norm2(lambda v: Rl @ v, lambda v: Rl.T @ v, n)
    del Rl
    t0 = time.time()
    Rb = _sn(hh.qr_blocked(A, nb=128)[1])
    print(f"c5: reference qr_blocked {time.time() - t0:.0f}s", flush=True)
    out["ref_diag"] = np.diag(Rb).copy()
    out["ref_rows"] = Rb[C5_ROWS].copy()
    out["ref_Rx"] = Rb @ x
    eps = np.finfo(float).eps
    print("c5: reference vs LAPACK rows: %.2f eps*||A||_2" %
          (np.max(np.abs(out["ref_rows"] - out["lapack_rows"])) / out["norm2"] / eps), flush=True)
    np.savez_compressed(os.path.join(OUT, "fullsize_c5.npz"), **out)


def states_fixture():
    """Philox state at every generation chunk of C3 / C4 / C5, so tests and
    bench.py regenerate the full inputs on a thread pool (fullsize.parallel_chunks)."""
    out = {}
    for cfg in ("c3", "c4", "c5"):
        st = []
        sha = fullsize.Sha()
        for _, blk in fullsize.chunks(cfg, states=st):
            sha.update(blk)
        out[f"{cfg}_states"] = np.stack(st)
        out[f"{cfg}_sha256"] = sha.hexdigest()
        print(cfg, len(st), "chunks", sha.hexdigest()[:16], flush=True)
    np.savez_compressed(os.path.join(OUT, "fullsize_states.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c2", "c4", "c3", "c5", "states"]
    for cfg in which:
        if cfg == "states":
            states_fixture()
        elif cfg == "c5":
            c5_fixture()
        else:
            tsqr_fixture(cfg)
