#!/usr/bin/env python
"""TSQR / CAQR benchmark on B200 (driver contract).

Default workload (N=1): BASELINE config 3, TSQR fp64 of A 16777216 x 128
iid N(0,1) (16 GiB, larger than L2), leaf blocks of 8192 x 128 + binary tree,
R only.  One "step" = one full TSQR of A resident in HBM.

  python bench.py                       # N=1, C3, R only
  python bench.py --config c4           # other configs (c1..c5)
  torchrun --nproc-per-node N bench.py --gpus N   # 1-D shards + cross-GPU tree
  python bench.py --impl reference      # the reference's CPU path (oracle port)

Metric: GFLOP/s with the standard Householder count F = 2mn^2 - 2n^3/3
(whole job).  ``roofline`` reports the leaf kernel against the FP64 peak,
``cpu_baseline`` the oracle port of the reference path on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.22
# DRAM bytes (read + write) over the 8mn algorithmic bytes, from this round's
# ncu --set full captures (profiles/r02/*_ncu_summary.txt)
NARROW8_TRAFFIC = (8.592664e9 + 3.943936e6) / (8 * 134217728 * 8)  # ncu dram read + write / 8mn, profiles/r02/narrow8_kernel_ncu_summary.txt
# k_leaf_tt<64, 1, false> at C3 full size, profiles/r02/leaf_tt_kernel_ncu_summary.txt
DMMA_TRAFFIC = (17.376649e9 + 7.044608e6) / (8.0 * 16777216 * 128)
METRIC = "TSQR fp64 GFLOP/s & % of roofline"

CONFIGS = {
    "c1": dict(key="c1", m=65536, n=32, leaf=8192, q="explicit", dist="normal",
               name="C1 TSQR 65536x32 N(0,1), 8 leaves of 8192, R + explicit Q"),
    "c2": dict(key="c2", m=1048576, n=64, leaf=4096, q="explicit", dist="cond",
               name="C2 TSQR 1048576x64 kappa=1e12, leaves of 4096, R + explicit Q"),
    "c3": dict(key="c3", m=16777216, n=128, leaf=8192, q="none", dist="normal",
               name="C3 TSQR 16777216x128 N(0,1), leaves of 8192x128, R only"),
    "c4": dict(key="c4", m=134217728, n=8, leaf=16384, q="none", dist="uniform",
               name="C4 TSQR 134217728x8 U(-1,1), leaves of 16384x8, R only"),
    "c5": dict(key="c5", m=16384, n=16384, leaf=2048, q="implicit", dist="normal",
               name="C5 CAQR 16384x16384 N(0,1), b=128, TSQR leaf 2048, R + implicit Q"),
}


def flops(m, n):
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def env_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------
def make_input(cfg, device, lo=0, hi=None, data="reference", seed=0):
    """Rows [lo, hi) of the config's input on ``device``.

    data = "reference" (default): the reference's own generators, bit for bit
    (rng_for(0) Philox draws, gen_cond_matrix for C2; paper_0809_2407_b200.synth
    regenerates any row range from recorded Philox states, so every rank draws
    only its shard).  data = "torch": torch Philox on the device (fast, for
    quick runs; not the reference's bits)."""
    import torch

    hi = cfg["m"] if hi is None else hi
    if data == "reference":
        from paper_0809_2407_b200 import synth

        return synth.device_input(cfg["key"], device, lo, hi)
    n = cfg["n"]
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if cfg["dist"] == "uniform":
        return torch.rand((hi - lo, n), generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0
    if cfg["dist"] == "cond":
        from paper_0809_2407_b200.core import CondSpec, gen_cond_matrix

        return torch.from_numpy(gen_cond_matrix(CondSpec(hi - lo, n, kappa=1e12, seed=seed))).to(device)
    return torch.randn((hi - lo, n), generator=g, dtype=torch.float64, device=device)


def host_sample(cfg, rows):
    """The first ``rows`` rows of the config's reference input, on the host."""
    from paper_0809_2407_b200 import synth

    out = np.empty((rows, cfg["n"]))

    def sink(r0, blk):
        out[r0:r0 + blk.shape[0]] = blk

    synth.chunks(cfg["key"], 0, rows, sink)
    return out


def _runs(m, P, n, q):
    """(chains, rows per chain) of the R-only leaf kernels on one GPU: csrc/tsqr_sm100.cu
    r_binary_impl deals the rows to at most CAQR_TUNE_FUSE = 148 CTAs in whole 64-row tiles
    (64 < n <= 128), or to 148 x 8 warps in whole 256-row steps (n <= 8)."""
    fuse, base = 148, m // P
    if q == "none" and (64 < n <= 128 or n <= 8):
        W, g = (fuse, 64) if n > 8 else (8 * fuse, 256)
        b2 = max(128, -(-(-(-m // W)) // g) * g)
        if P > W and b2 > base:
            P2 = -(-m // b2)
            if P2 > 1 and m - (P2 - 1) * b2 < n:
                P2 -= 1
            return P2, b2
    return P, base


def _tree_note(m, P, n, q):
    """How the rows of one GPU are combined (CAQR_TUNE_FUSE, csrc/tsqr_sm100.cu r_binary_impl)."""
    P2, b2 = _runs(m, P, n, q)
    if P2 != P:
        who = "a CTA" if n > 8 else "a warp"
        unit = "64-row tiles" if n > 8 else "256-row steps"
        return (f"flat tree inside {who} over runs of {b2} rows ({P2} runs, whole {unit}), "
                "binary tree above (hybrid tree, PAPER.md Fig. 3); CAQR_TUNE=16=0 gives the binary tree "
                "over all leaves")
    return "binary tree over the leaves"


def parity_vs_reference(cfg, R):
    """The timed run's R against the reference's R on the same input
    (tests/golden/fullsize_<cfg>.npz, made by oracle/make_fullsize.py from the
    read-only reference): max |sn(R) - sn(R_ref)| in eps ||A||_2, bar 1000
    (pkg/tests/test_householder.py:340-350).  None when the fixture is absent."""
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{cfg['key']}.npz")
    if R is None or not os.path.exists(path):
        return None
    f = np.load(path)
    Rn = R.detach().cpu().numpy() if hasattr(R, "detach") else np.asarray(R)
    eps = float(np.finfo(np.float64).eps)

    def sn(X):
        d = np.sign(np.diag(X)).copy()
        d[d == 0] = 1.0
        return d[:, None] * X

    if cfg["key"] == "c5":
        d = np.sign(np.diag(Rn)).copy()
        d[d == 0] = 1.0
        rows = f["rows"]
        err = max(float(np.max(np.abs(d[rows, None] * Rn[rows] - f["ref_rows"]))),
                  float(np.max(np.abs(d * np.diag(Rn) - f["ref_diag"]))))
        err /= float(f["norm2"]) * eps
        what = "reference qr_blocked(A, 128): sign-normalised diagonal + 8 rows"
    else:
        err = float(np.max(np.abs(sn(Rn) - sn(f["R_ref"])))) / (float(f["norm2"]) * eps)
        what = "reference Alg. 1 composition (qr_unblocked leaves + qr_stacked_triangles tree)"
    return {"vs": what, "fixture": os.path.relpath(path, ROOT), "r_err_eps_norm2": err,
            "bar": 1000.0, "ok": bool(err <= 1000.0)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference path (oracle port) on a bounded sample
# ---------------------------------------------------------------------------
_POOL_A = None  # the sample the forked leaf workers read (copy-on-write)


def _pool_init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        pass


def _pool_leaf(args):
    import oracle

    i, leaf = args
    return oracle.geqr2(_POOL_A[i * leaf:(i + 1) * leaf])[2]


def cpu_baseline_procs(cfg, budget_s, procs):
    """The reference path with its leaves spread over `procs` forked worker processes (one BLAS
    thread each): TSQR's leaves are independent, so this is the reference's algorithm using all
    the host cores; the tree over the leaf R factors runs in the parent."""
    import multiprocessing as mp

    import oracle

    global _POOL_A
    n, leaf = cfg["n"], min(cfg["leaf"], cfg["m"])
    t0 = time.perf_counter()
    oracle.geqr2(host_sample(cfg, leaf))
    t_leaf = time.perf_counter() - t0
    cap = max(procs, (1 << 30) // (8 * leaf * n))  # at most 1 GiB of sample
    nleaves = min(int(budget_s * procs / max(t_leaf, 1e-3)), cap) // procs * procs
    nleaves = max(2, min(max(nleaves, procs), cfg["m"] // leaf))
    _POOL_A = host_sample(cfg, nleaves * leaf)
    with mp.get_context("fork").Pool(procs, initializer=_pool_init) as pool:
        pool.map(_pool_leaf, [(i, leaf) for i in range(min(procs, nleaves))])  # workers up, pages touched
        t0 = time.perf_counter()
        Rs = pool.map(_pool_leaf, [(i, leaf) for i in range(nleaves)], chunksize=1)
        for (lvl, a, b) in oracle.binary_events(nleaves):
            _, _, Rs[a] = oracle.stacked_qr(Rs[a], Rs[b])
        dt = time.perf_counter() - t0
    _POOL_A = None
    m_s = nleaves * leaf
    return {"value": flops(m_s, n) / dt / 1e9, "unit": "GFLOP/s",
            "sample": (f"reference path (geqr2 leaves over {procs} worker processes + stacked_qr binary tree), "
                       f"the first {nleaves} leaves of {leaf}x{n} of the config input = {m_s} rows, R only"
                       + ("; Q not formed in the sample" if cfg["q"] != "none" else "")),
            "seconds": dt}


def cpu_baseline(cfg, budget_s=15.0, threads=None):
    import oracle

    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    n = cfg["n"]
    leaf = min(cfg["leaf"], cfg["m"])
    ctx = threadpool_limits(limits=threads) if (threadpool_limits and threads) else None
    if ctx:
        ctx.__enter__()
    try:
        if cfg is CONFIGS["c5"]:
            N = 2048
            A = host_sample(cfg, N)[:, :N].copy()  # leading 2048 x 2048 block of the C5 input
            t0 = time.perf_counter()
            oracle.blocked_qr(A, 128)
            dt = time.perf_counter() - t0
            return {"value": flops(N, N) / dt / 1e9, "unit": "GFLOP/s",
                    "sample": f"reference qr_blocked(A, nb=128) on the leading {N}x{N} block "
                              f"of the C5 input (C5 scaled 1/8)", "seconds": dt}
        # one leaf first to size the sample; leaves are the config input's first rows
        Aleaf = host_sample(cfg, leaf)
        t0 = time.perf_counter()
        Y, tau, R = oracle.geqr2(Aleaf)
        t_leaf = time.perf_counter() - t0
        Rs = [R]
        t_comb = 0.0
        nleaves = max(2, min(int(budget_s / max(t_leaf, 1e-3)), cfg["m"] // leaf))
        Asamp = host_sample(cfg, nleaves * leaf)
        t0 = time.perf_counter()
        for i in range(1, nleaves):
            Y, tau, R = oracle.geqr2(Asamp[i * leaf:(i + 1) * leaf])
            Rs.append(R)
        t_rest = time.perf_counter() - t0
        t0 = time.perf_counter()
        for (lvl, a, b) in oracle.binary_events(nleaves):
            _, _, Rs[a] = oracle.stacked_qr(Rs[a], Rs[b])
        t_comb = time.perf_counter() - t0
        dt = t_leaf + t_rest + t_comb
        m_s = nleaves * leaf
        q = cfg["q"] != "none"
        return {"value": flops(m_s, n) / dt / 1e9, "unit": "GFLOP/s",
                "sample": (f"reference path (geqr2 leaves + stacked_qr binary tree), the first "
                           f"{nleaves} leaves of {leaf}x{n} of the config input = {m_s} rows, R only"
                           + ("; Q not formed in the sample" if q else "")),
                "seconds": dt}
    finally:
        if ctx:
            ctx.__exit__(None, None, None)


def run_reference(args, cfg):
    ws, rank, _ = env_dist()
    if rank != 0:
        return
    ncpu = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        budget = max(2.0, 60.0 / max(1, args.steps + args.warmup))
        if cfg is CONFIGS["c5"] or ncpu < 2:
            cb = cpu_baseline(cfg, budget_s=budget, threads=ncpu)  # BLAS-3 blocked QR: BLAS threads
        else:
            cb = cpu_baseline_procs(cfg, budget_s=budget, procs=ncpu)
        if i >= args.warmup:
            vals.append(cb)
    v = float(np.median([c["value"] for c in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.median([c["seconds"] for c in vals]) * 1e3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's generators (rng_for(0) / gen_cond_matrix), the same "
                "bits as the GPU arm's input",
        "config": {"workload": cfg["name"], "m": cfg["m"], "n": cfg["n"], "leaf_rows": cfg["leaf"]},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": ncpu, "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our path
# ---------------------------------------------------------------------------
def caqr_roofline(A, cfg, args):
    """Roofline of CAQR's dominant kernel, the leaf-level trailing update
    (k_leaf_apply, Q_0^T applied to the n - b trailing columns of panel 0):
    4 m b (n - b) algorithmic flops per launch over its event-timed duration.
    Also returns the number of library kernels one caqr_factor launches."""
    from paper_0809_2407_b200.caqr import _panel_leaves, caqr_factor
    import torch

    from paper_0809_2407_b200.tsqr import _leaf_apply, factor_device

    m, n = A.shape
    b = 128
    full = caqr_factor(A, b=b, leaf_rows=cfg["leaf"], panel_chains=args.panel_chains, apply_waves=args.apply_waves)
    launches = full.launches
    del full
    P = _panel_leaves(m, b, cfg["leaf"])
    f = factor_device(A[:, :b].contiguous(), P, want_q=True)
    C = A[:, b:].contiguous()
    for _ in range(2):
        _leaf_apply(f, C, transpose=True)
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _leaf_apply(f, C, transpose=True)
        e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    t = float(np.mean([a.elapsed_time(c) for a, c in ts])) * 1e-3
    F = 4.0 * m * b * (n - b)
    ach = F / t / 1e12
    del C, f
    torch.cuda.empty_cache()
    return ({"bound": "fp64", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
             "frac": ach / FP64_PEAK_TFLOPS, "traffic": None,
             "kernel": "k_leaf_apply (trailing update of panel 0: Q_0^T on m x (n-b))",
             "peak_source": "148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (BASELINE.md; no FP64 "
                            "entry in MEASURED_PEAKS.json)",
             "algorithmic_flops_per_launch": F, "launch_ms": t * 1e3}, launches)


def data_note(cfg, args):
    if args.data == "reference":
        return ("synthetic: the reference's own generators, bit for bit (" +
                ("gen_cond_matrix(CondSpec(2**20, 64, 1e12, 0)), pinned BLAS" if cfg["key"] == "c2"
                 else "rng_for(0) Philox draws, " + cfg["dist"]) +
                "; each rank regenerates its row shard; paper_0809_2407_b200.synth)")
    return "synthetic iid " + cfg["dist"] + " (torch Philox on device, seed = rank)"


def run_grid(args, cfg, ws, rank, local):
    """C5 on a 2 x (N/2) process grid (Algorithm 3, paper_0809_2407_b200.grid):
    block-cyclic 128 x 128 blocks, one rank per GPU, NCCL row / column groups.
    Every rank generates the same seeded A and keeps its own blocks."""
    import torch
    import torch.distributed as dist

    from paper_0809_2407_b200.core import BlockCyclicLayout
    from paper_0809_2407_b200.grid import GpuBackend, caqr_grid, gather_R, make_grid, scatter_local

    dev = torch.device("cuda", local)
    m, n, b = cfg["m"], cfg["n"], 128
    Pr = 2 if ws % 2 == 0 else 1  # C5: 2 x 4 at 8 GPUs
    Pc = ws // Pr
    grid = make_grid(BlockCyclicLayout(m, n, b, Pr, Pc))
    A = make_input(cfg, dev, data=args.data)
    base = scatter_local(A, grid)
    del A
    be = GpuBackend(leaf_rows=cfg["leaf"])
    work = torch.empty_like(base)
    stream = torch.cuda.current_stream(dev)

    def step():
        work.copy_(base)
        return caqr_grid(work, grid, be, lookahead=args.grid_lookahead)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    copy_ms = 0.0
    with Clocks(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        dist.barrier()
        torch.cuda.synchronize()
    # the per-step reset copy of the local blocks is not CAQR work: time it alone
    c0 = torch.cuda.Event(enable_timing=True)
    c1 = torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(args.steps):
        work.copy_(base)
    c1.record(stream)
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(c1) / args.steps
    ms = t0.elapsed_time(t1) / args.steps - copy_ms
    ms_t = torch.tensor([ms], device=dev)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    F = flops(m, n)
    value = F / (ms * 1e-3) / 1e9
    e2e = None
    if not args.no_e2e:
        # host blocks (pinned) -> device, Algorithm 3, R gathered back to rank 0's host
        hostb = torch.empty(base.shape, dtype=torch.float64, pin_memory=True)
        hostb.copy_(base)
        dist.barrier()
        ts = time.perf_counter()
        loc = hostb.to(dev, non_blocking=True)
        R = gather_R(caqr_grid(loc, grid, be))
        Rh = R.cpu() if R is not None else None
        dist.barrier()
        dt = time.perf_counter() - ts
        dt_t = torch.tensor([dt], device=dev)
        dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
        dt = float(dt_t.item())
        e2e = {"value": F / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(m * n * 8),
               "d2h_bytes_per_step": int(n * n * 8), "ms_per_step": dt * 1e3}
        del Rh
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": data_note(cfg, args),
            "config": {"workload": cfg["name"] + f", {Pr}x{Pc} grid", "m": m, "n": n, "b": b,
                       "leaf_rows": cfg["leaf"], "parallelism": f"2-D block-cyclic {Pr}x{Pc}",
                       "l2": "inputs larger than L2 (no flush needed)",
                       "timing": "events around K steps minus the per-step block reset copy"},
            "roofline": None, "cpu_baseline": None, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": None, "gflops_roofline_frac": value / (FP64_PEAK_TFLOPS * 1e3 * ws),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import _leaves_for, explicit_q_device, factor_device

    ws, rank, local = env_dist()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.load()
    m, n = cfg["m"], cfg["n"]
    is_caqr = cfg is CONFIGS["c5"]
    if is_caqr and (ws > 1 or args.grid):
        if not dist.is_initialized():  # --grid on one GPU: a 1 x 1 grid
            import socket

            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                    world_size=1, device_id=torch.device("cuda", local))
        return run_grid(args, cfg, ws, rank, local)
    # shard rows (1-D block rows); A resident in HBM
    from paper_0809_2407_b200.dist import shard_rows, tsqr_sharded

    lo, hi = shard_rows(m, ws, rank)
    A = (make_input(cfg, dev, lo, hi, data=args.data, seed=rank) if not is_caqr
         else make_input(cfg, dev, data=args.data))
    P = _leaves_for(hi - lo, n, cfg["leaf"])
    from paper_0809_2407_b200.tsqr import split_leaves

    chains = 1 if is_caqr else split_leaves(hi - lo, n, P, fill=(n > 8 and cfg["q"] == "none"),
                                                  narrow=(n <= 8 and cfg["q"] == "none"))
    P *= chains
    want_q = cfg["q"] != "none"
    stream = torch.cuda.current_stream(dev)

    leaf_ev = []
    last = {}

    def step(record=False):
        if is_caqr:
            from paper_0809_2407_b200.caqr import caqr_factor

            last["f"] = caqr_factor(A, b=128, leaf_rows=cfg["leaf"], panel_chains=args.panel_chains, apply_waves=args.apply_waves)
            return last["f"]
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        f = factor_device(A, P, want_q=want_q)
        last["f"] = f
        if record:
            e1.record(stream)
            leaf_ev.append((e0, e1))
        if ws > 1:
            # cross-GPU binary tree of the per-rank R factors; explicit Q walks
            # back down it (dist.tsqr_sharded_explicit_q)
            from paper_0809_2407_b200.dist import cross_tree, gpu_combine, tsqr_sharded_explicit_q

            _, nodes = cross_tree(f.R, gpu_combine)
            if cfg["q"] == "explicit":
                tsqr_sharded_explicit_q(f, nodes)
            return f
        if cfg["q"] == "explicit":
            explicit_q_device(f)
        return f

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    leaf_ev.clear()
    graph = None
    if args.graph and not is_caqr and ws == 1:
        # capture one whole step (every kernel of the factorization and of the
        # Q formation) in a CUDA graph; the NaN/Inf flag is checked after replay
        g_stream = torch.cuda.Stream(device=dev)
        g_stream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(g_stream):
            holder = {}

            def gstep():
                f = factor_device(A, P, want_q=want_q, check=False)
                holder["f"] = f
                if cfg["q"] == "explicit":
                    holder["q"] = explicit_q_device(f)

            gstep()  # allocate the pool outside capture
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=g_stream):
                gstep()
        stream.wait_stream(g_stream)
        torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        t0.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step(record=not is_caqr)
        t1.record(stream)
        barrier()
    if graph is not None:
        holder["f"].check_finite()
        # the graph replays bracket the same kernels; time them for the roofline
        for _ in range(2):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            leaf_ev.append((e0, e1))
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    F = flops(m, n)
    value = F / (ms * 1e-3) / 1e9
    # parity of the timed computation's R against the reference's R on the same input
    R_timed = None
    if graph is not None:
        R_timed = holder["f"].R_out()
    elif is_caqr:
        R_timed = last["f"].R if last else None
    elif last:
        f_last = last["f"]
        if ws > 1:
            from paper_0809_2407_b200.dist import cross_tree, gpu_combine

            R_timed, _ = cross_tree(f_last.R, gpu_combine)
        else:
            R_timed = f_last.R_out()
    parity = parity_vs_reference(cfg, R_timed) if (rank == 0 and args.data == "reference") else None
    del R_timed

    # roofline of the dominant kernel: the leaf factorization (factor_device's
    # leaf + tree events bracket; the tree is < 2% of it, see profiles/)
    roof = None
    caqr_launches = None
    if is_caqr:
        detail, caqr_launches = caqr_roofline(A, cfg, args)
        ach = F / (ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP64_PEAK_TFLOPS, "traffic": None,
                "kernel": "the whole CAQR step (panel TSQRs, leaf- and tree-level trailing updates, "
                          "two-stream lookahead): F = 2mn^2 - 2n^3/3 over ms_per_step",
                "peak_source": detail["peak_source"], "algorithmic_flops_per_launch": F,
                "detail_panel0_trailing_update": {k: detail[k] for k in
                                                  ("kernel", "achieved", "frac", "launch_ms",
                                                   "algorithmic_flops_per_launch")}}
    if leaf_ev:
        # the timed bracket: one factor_device call (or the graph replay of the
        # step, which for explicit-Q configs also forms Q: 2x the flops)
        t_leaf = float(np.mean([a.elapsed_time(b) for a, b in leaf_ev])) * 1e-3
        qmul = 2 if cfg["q"] == "explicit" else 1
        F_leaf = qmul * flops(hi - lo, n)
        hbm = 6526.5
        try:
            hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            pass
        t_flop = F_leaf / (FP64_PEAK_TFLOPS * 1e12)
        t_byte = 8.0 * (hi - lo) * n / (hbm * 1e9)
        narrow = n <= 8 and cfg["q"] == "none"
        if cfg["q"] == "none" and t_byte > t_flop:
            # HBM-bound (C4, AI = n/4 flop/B < the 5.7 ridge): bytes of A per launch
            ach = 8.0 * (hi - lo) * n / t_leaf / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": 8.0 * (hi - lo) * n * NARROW8_TRAFFIC if narrow else None,
                    "traffic_source": "ncu --set full of k_leaf_narrow8 (profiles/r02/"
                                      "narrow8_kernel_ncu_summary.txt): dram read + write = "
                                      f"{NARROW8_TRAFFIC:.4f} x 8mn, scaled per launch",
                    "kernel": "k_leaf_narrow8 (8 rows per reflector chain) + fused ticket tree "
                              "(one factor_device call)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "algorithmic_bytes_per_launch": 8.0 * (hi - lo) * n}
        else:
            ach = F_leaf / t_leaf / 1e12
            # DRAM traffic of the leaf kernel from the committed ncu capture
            # (profiles/r02/leaf_tt_kernel_ncu_summary.txt: 17.377 GB read + 7.0 MB
            # written at C3 full size = 1.0119x the 8mn algorithmic bytes), scaled
            # to this launch's rows; None for other widths.
            traffic = 8.0 * (hi - lo) * n * DMMA_TRAFFIC if (n == 128 and cfg["q"] == "none") else None
            kern = (("k_leaf_tt<64,1> (tall tiles in tensor memory, CTAs chaining consecutive leaves) + "
                     "k_tree_ring (one factor_device call)" if n > 64 else
                     "k_leaf_dmma (DMMA warp ring) + k_tree_ring (one factor_device call)")
                    if cfg["q"] == "none" else
                    ("k_leaf_dense + k_leaf_dmma<64> + k_tree_factor_dmma, then Q: k_tree_apply_dmma + "
                     "k_leaf_q_dmma<64> " if 32 < n <= 64 else
                     "k_leaf_dense + k_leaf_chain + k_tree_factor_dmma, then Q: k_tree_apply_dmma + "
                     "k_leaf_q_dmma<32> ") +
                    "(graph replay of the step; credited with the factor and Q-formation flops)")
            roof = {"bound": "fp64", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP64_PEAK_TFLOPS, "traffic": traffic,
                    "traffic_source": "ncu --set full of k_leaf_tt at C3 full size, profiles/r02/leaf_tt_kernel_ncu_summary.txt (scaled per launch)",
                    "kernel": kern,
                    "peak_source": "148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (BASELINE.md; no FP64 "
                                   "entry in MEASURED_PEAKS.json)",
                    "algorithmic_flops_per_launch": F_leaf}
        if cfg["q"] == "none":
            t_roof = max(t_flop, t_byte)
            roof["t_roof_ms"] = t_roof * 1e3
            roof["roofline_frac_time"] = t_roof / t_leaf

    # e2e through the public API with host buffers (pinned), rank 0 view
    e2e = None
    if not args.no_e2e:
        from paper_0809_2407_b200.tsqr import tsqr

        Ah = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
        Ah.copy_(A)
        e_steps = max(1, min(args.steps, 3))
        if is_caqr:
            from paper_0809_2407_b200.caqr import caqr_factor

            def e2e_step():
                res = caqr_factor(Ah, b=128, leaf_rows=cfg["leaf"], panel_chains=args.panel_chains, apply_waves=args.apply_waves)
                return res.R
        elif ws == 1:
            def e2e_step():
                out = tsqr(Ah, leaf_rows=cfg["leaf"], q=cfg["q"])
                return out
        else:
            from paper_0809_2407_b200.dist import cross_tree, gpu_combine, tsqr_sharded_explicit_q

            def e2e_step():
                # this rank's shard from pinned host memory -> local TSQR (streamed
                # when R only) -> cross-GPU tree -> R (and this rank's Q rows) to host
                if cfg["q"] == "none":
                    Rl = torch.from_numpy(tsqr(Ah, leaf_rows=cfg["leaf"])).to(dev)
                    R, _ = cross_tree(Rl, gpu_combine)
                    return None if R is None else R.cpu()
                _, f = tsqr(Ah, leaf_rows=cfg["leaf"], q="implicit")
                R, nodes = cross_tree(f.R, gpu_combine)
                Q = tsqr_sharded_explicit_q(f, nodes).cpu()
                return Q, (None if R is None else R.cpu())
        # two warm-up calls: results alternate between two host buffers, so the
        # caching pinned allocator is in steady state before timing
        out = e2e_step()
        out = e2e_step()
        barrier()
        ts = time.perf_counter()
        for _ in range(e_steps):
            out = e2e_step()
        barrier()
        dt = (time.perf_counter() - ts) / e_steps
        d2h = n * n * 8 + (m * n * 8 if cfg["q"] == "explicit" else 0)
        if is_caqr:
            d2h = n * n * 8
        e2e_v = F / dt / 1e9
        dt_t = torch.tensor([dt], device=dev)
        if ws > 1:
            dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
            e2e_v = F / float(dt_t.item()) / 1e9
        e2e = {"value": e2e_v, "unit": "GFLOP/s", "h2d_bytes_per_step": int(A.numel() * 8) * ws,
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(dt_t.item()) * 1e3}
        del Ah

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cb = cpu_baseline(cfg, budget_s=args.cpu_budget, threads=1)
        cpu = {"value": cb["value"], "unit": "GFLOP/s", "cores": 1, "kind": "port",
               "sample": cb["sample"]}
    P_run = _runs(hi - lo, P, n, cfg["q"])[0]
    levels = max(0, int(np.ceil(np.log2(P_run)))) if P_run > 1 else 0
    launches = (1 + levels) * args.steps
    if n <= 8 and cfg["q"] == "none":
        launches = args.steps  # leaf kernel with the ticket tree fused (one kernel per step)
    if cfg["q"] == "explicit":
        launches += (levels + 1) * args.steps
    if is_caqr:
        launches = caqr_launches * args.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": data_note(cfg, args),
            "config": {"workload": cfg["name"], "m": m, "n": n, "leaf_rows": cfg["leaf"],
                       "leaves_per_gpu": P // chains, "gpu_chains_per_leaf": chains, "outputs": cfg["q"], "parallelism": f"1-D rows x{ws}",
                       "l2": "inputs larger than L2 (no flush needed)" if 8 * m * n > 256e6
                       else "inputs smaller than L2",
                       "tree": _tree_note(hi - lo, P, n, cfg["q"])},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
            "clocks": clk.summary(), "gpu_launches": launches,
            "cuda_graph": graph is not None,
            "gflops_roofline_frac": value / (FP64_PEAK_TFLOPS * 1e3 * ws),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--graph", type=int, default=1,
                    help="replay each TSQR step as one captured CUDA graph (1 GPU, not CAQR)")
    ap.add_argument("--grid", action="store_true",
                    help="c5: run the Pr x Pc grid driver even on one GPU (1 x 1 grid)")
    ap.add_argument("--data", default="reference", choices=["reference", "torch"],
                    help="inputs: the reference's generators bit for bit (default) or torch Philox")
    ap.add_argument("--grid-lookahead", action="store_true", help="c5 grid: two-stream lookahead")
    ap.add_argument("--apply-waves", type=float, default=4.0, help="c5: waves of trailing-update CTAs per panel")
    ap.add_argument("--panel-chains", type=int, default=4,
                    help="CAQR: split each panel's leaves into GPU chains up to this count")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
