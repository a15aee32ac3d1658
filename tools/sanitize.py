"""One small invocation of every hand-written kernel with a synchronisation
protocol (warp rings with acquire/release counters, named barriers, ticket
trees), for compute-sanitizer (racecheck / synccheck / memcheck), CI sizes:

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.caqr import caqr_apply_q, caqr_factor
from paper_0809_2407_b200.householder import form_t, qr_unblocked
from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

rng = np.random.Generator(np.random.Philox(7))


def dev(a):
    return torch.from_numpy(a).cuda()


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


A128 = dev(rng.standard_normal((2048 + 256, 128)))
A64 = dev(rng.standard_normal((2048, 64)))
A32 = dev(rng.standard_normal((1024, 32)))
A8 = dev(rng.uniform(-1, 1, (16384 * 2 + 300, 8)))
run("k_leaf_dmma<128> R only + k_tree_ring", lambda: factor_device(A128, 2))
run("k_leaf_dense + k_leaf_dmma<128, Q> + k_tree_factor<128>", lambda: factor_device(A128, 2, want_q=True))
run("k_leaf_q_dmma<128> + k_tree_apply_dmma (explicit Q)",
    lambda: explicit_q_device(factor_device(A128, 2, want_q=True)))
run("NP = 64 ring + k_tree_factor_dmma<64> + k_leaf_q_dmma<64>",
    lambda: explicit_q_device(factor_device(A64, 2, want_q=True)))
run("k_leaf_chain<32> + k_tree_factor_dmma<32> + k_leaf_q_dmma<32>",
    lambda: explicit_q_device(factor_device(A32, 4, want_q=True)))
run("k_leaf_narrow8 + fused ticket tree", lambda: factor_device(A8, 2))
_lib.tune(_lib.TUNE_NARROW, 2)
run("k_leaf_narrow<cp.async, K=4> + fused ticket tree", lambda: factor_device(A8, 2))
_lib.reset_tuning()
_lib.tune(_lib.TUNE_CC, 2)
run("k_leaf_split (generation + update warps)", lambda: factor_device(A128, 2))
_lib.reset_tuning()
C = dev(rng.standard_normal((1024, 384)))
run("caqr_factor: k_leaf_apply_dmma + k_tree_apply_dmma (lookahead streams)",
    lambda: caqr_apply_q(caqr_factor(C, b=128, leaf_rows=512), C[:, :3].contiguous()))
B = rng.standard_normal((300, 150))
run("k_geqr2 + k_form_t", lambda: form_t(qr_unblocked(B)[0].Y, qr_unblocked(B)[0].tau))
print("sanitize: all kernels ran")
