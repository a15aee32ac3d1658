"""Generate tests/golden/*.npz by running the READ-ONLY reference itself.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py

The reference package has no ``__init__.py`` and its name collides with the
drop-in package ``caqr`` of this repo, so it is imported under the alias
``caqr_ref``.  Nothing here is copied from the
reference: the script only calls its public functions and stores their
outputs as small fixtures, which the CPU tests compare with the oracle
restatement and the GPU tests compare with the CUDA path.
"""

from __future__ import annotations

import importlib
import os
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src/caqr"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def load_reference():
    if "caqr_ref" not in sys.modules:
        pkg = types.ModuleType("caqr_ref")
        pkg.__path__ = [REF]
        sys.modules["caqr_ref"] = pkg
    mods = {}
    for name in ("core", "householder", "trees", "counters"):
        mods[name] = importlib.import_module(f"caqr_ref.{name}")
    return mods


def main():
    ref = load_reference()
    core, hh, trees = ref["core"], ref["householder"], ref["trees"]
    os.makedirs(OUT, exist_ok=True)

    # ---- dense leaf QR (householder.py:128) on seeded inputs -------------
    kernels = {}
    for (m, n, seed) in [(6, 3, 7), (40, 8, 1), (96, 32, 2), (160, 64, 3)]:
        A = core.rng_for(seed).standard_normal((m, n))
        f, R = hh.qr_unblocked(A)
        kernels[f"unb_{m}x{n}_A"] = A
        kernels[f"unb_{m}x{n}_Y"] = f.Y
        kernels[f"unb_{m}x{n}_tau"] = f.tau
        kernels[f"unb_{m}x{n}_R"] = R
        kernels[f"unb_{m}x{n}_T"] = hh.form_t(f.Y, f.tau)
        kernels[f"unb_{m}x{n}_Q"] = hh.explicit_q(f)
    # ---- stacked triangles q = 2 (householder.py:263) ---------------------
    for (n, seed) in [(5, 30), (8, 31), (32, 32), (64, 33)]:
        rng = core.rng_for(seed)
        Ra = np.triu(rng.standard_normal((n, n)))
        Rb = np.triu(rng.standard_normal((n, n)))
        f, R = hh.qr_stacked_triangles([Ra, Rb])
        kernels[f"stk_{n}_Ra"] = Ra
        kernels[f"stk_{n}_Rb"] = Rb
        kernels[f"stk_{n}_Y"] = f.Y
        kernels[f"stk_{n}_tau"] = f.tau
        kernels[f"stk_{n}_R"] = R
        C = rng.standard_normal((2 * n, 3))
        kernels[f"stk_{n}_C"] = C
        kernels[f"stk_{n}_QC"] = hh.apply_q(f, C)
        kernels[f"stk_{n}_QtC"] = hh.apply_qt(f, C)
    # ---- triangle on rectangle (householder.py:297) -----------------------
    for (n, r, seed) in [(5, 7, 42), (8, 16, 43), (32, 32, 44), (64, 40, 45)]:
        rng = core.rng_for(seed)
        R0 = np.triu(rng.standard_normal((n, n)))
        B = rng.standard_normal((r, n))
        f, R = hh.qr_triangle_on_rect(R0, B)
        kernels[f"tor_{n}x{r}_R0"] = R0
        kernels[f"tor_{n}x{r}_B"] = B
        kernels[f"tor_{n}x{r}_Y"] = f.Y
        kernels[f"tor_{n}x{r}_tau"] = f.tau
        kernels[f"tor_{n}x{r}_R"] = R
        C = rng.standard_normal((n + r, 2))
        kernels[f"tor_{n}x{r}_C"] = C
        kernels[f"tor_{n}x{r}_QC"] = hh.apply_q(f, C)
        kernels[f"tor_{n}x{r}_QtC"] = hh.apply_qt(f, C)
        T = hh.factor_t(f)
        C0, C1 = hh.apply_qt_structured(f, T, C[:n], C[n:])
        kernels[f"tor_{n}x{r}_T"] = T
        kernels[f"tor_{n}x{r}_S0"] = C0
        kernels[f"tor_{n}x{r}_S1"] = C1
    # ---- blocked QR (householder.py:189), the CAQR Pr=Pc=1 degenerate -----
    A = core.rng_for(11).standard_normal((256, 128))
    f, R = hh.qr_blocked(A, nb=32)
    kernels["blk_256x128_A"] = A
    kernels["blk_256x128_R"] = R
    kernels["blk_256x128_tau"] = f.tau
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **kernels)

    # ---- composed TSQR with the reference kernels -----------
    comp = {}
    for (m, n, P, seed, kappa) in [(2048, 32, 8, 5, None), (1024, 64, 8, 6, 1e12),
                                   (1201, 16, 5, 7, None)]:
        if kappa is None:
            A = core.rng_for(seed).standard_normal((m, n))
        else:
            A = core.gen_cond_matrix(core.CondSpec(m, n, kappa=kappa, seed=seed))
        lay = core.BlockRowLayout(m, n, P)
        offs = lay.row_offsets()
        blocks = core.partition_block_rows(A, P)
        facs, Rs = [], []
        for blk in blocks:
            fl, Rl = hh.qr_unblocked(blk)
            facs.append(fl)
            Rs.append(Rl)
        tree = trees.ReductionTree(P=P, shape="binary")
        nodes = []
        for ev in tree.schedule():
            a, b = ev.participants
            fn, Rn = hh.qr_stacked_triangles([Rs[a], Rs[b]])
            nodes.append((a, b, fn))
            Rs[a] = Rn
        S = [None] * P
        S[0] = np.eye(n)
        for (a, b, fn) in reversed(nodes):
            C = hh.apply_q(fn, np.vstack([S[a], np.zeros((n, n))]))
            S[a], S[b] = C[:n], C[n:]
        Q = np.zeros((m, n))
        for i, fl in enumerate(facs):
            C = np.zeros((offs[i + 1] - offs[i], n))
            C[:n] = S[i]
            Q[offs[i]:offs[i + 1]] = hh.apply_q(fl, C)
        tag = f"tsqr_{m}x{n}_P{P}"
        comp[f"{tag}_A"] = A
        comp[f"{tag}_R"] = Rs[0]
        comp[f"{tag}_Q"] = Q
        comp[f"{tag}_offs"] = np.array(offs)
    np.savez_compressed(os.path.join(OUT, "tsqr.npz"), **comp)

    # ---- trees and generators ---------------------------------------------
    misc = {}
    for P in (1, 2, 3, 4, 5, 8, 13, 16, 148, 2048):
        ev = trees.ReductionTree(P=P, shape="binary").schedule()
        misc[f"sched_{P}"] = np.array([(e.level,) + tuple(e.participants) for e in ev],
                                      dtype=np.int64).reshape(-1, 3)
    misc["cond_64x8_k1e12_s3"] = core.gen_cond_matrix(core.CondSpec(64, 8, kappa=1e12, seed=3))
    misc["normal_s0_1000x8"] = core.rng_for(0).standard_normal((1000, 8))
    misc["uniform_s0_1000x8"] = core.rng_for(0).uniform(-1, 1, (1000, 8))
    lay = core.BlockCyclicLayout(1024, 1024, 128, 2, 4)
    misc["bc_owner"] = np.array([[lay.owner(i, j) for j in range(8)] for i in range(8)])
    np.savez_compressed(os.path.join(OUT, "misc.npz"), **misc)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
