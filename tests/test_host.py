"""Host-side logic (no GPU): trees, layouts, generators, counters, the C-ABI
library's exported symbols, and the drop-in ``caqr`` package."""

import ctypes
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from paper_0809_2407_b200 import _lib
from paper_0809_2407_b200.core import (
    BlockCyclicLayout,
    BlockRowLayout,
    CondSpec,
    DimensionError,
    gen_cond_matrix,
    partition_block_rows,
    rng_for,
)
from paper_0809_2407_b200.counters import (
    CommRecorder,
    FlopCounter,
    count_geqr2,
    count_stacked,
    critical_path,
)
from paper_0809_2407_b200.trees import (
    ReductionTree,
    TreeError,
    build_qary_levels,
    first_proc,
    level,
    parse_tree,
    qary_tree,
    target_first_proc,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- trees (reference tests: pkg/tests/test_trees.py) ----------------------

def test_node_arithmetic():
    assert level(5, 0) == 5 and level(5, 2) == 1 and level(7, 3) == 0
    for i in range(4, 8):
        assert first_proc(i, 2) == 4 and target_first_proc(i, 2) == 6
    assert first_proc(3, 1) == 2 and target_first_proc(3, 1) == 3
    with pytest.raises(TreeError):
        target_first_proc(3, 0)


def test_schedules(golden):
    ev = ReductionTree(P=4).schedule()
    assert [(e.level, e.participants, e.receiver) for e in ev] == [
        (1, (0, 1), 0), (1, (2, 3), 2), (2, (0, 2), 0)]
    assert ReductionTree(P=1).schedule() == []
    assert [(e.participants, e.receiver) for e in ReductionTree(P=4, shape="flat").schedule()] == [
        ((0, 1), 0), ((0, 2), 0), ((0, 3), 0)]
    for k, v in golden["misc"].items():
        if k.startswith("sched_"):
            P = int(k.split("_")[1])
            got = np.array([(e.level,) + e.participants for e in ReductionTree(P=P).schedule()],
                           dtype=np.int64).reshape(-1, 3)
            assert np.array_equal(got, v), P


@given(st.integers(2, 64))
@settings(max_examples=40, deadline=None)
def test_binary_pairing(P):
    tree = ReductionTree(P=P)
    consumed = [p for grp in tree.levels for g in grp for p in g[1:]]
    assert sorted(consumed + [tree.root]) == list(range(P))
    lv = tree.device_levels()
    ids = np.concatenate([x[:, 2] for x in lv])
    assert list(ids) == list(range(P - 1))
    assert sum(len(x) for x in lv) == P - 1


def test_tree_misc():
    assert ReductionTree(P=16).critical_path_stats() == {"stages": 4, "messages_per_proc": 4}
    assert ReductionTree(P=4, shape="flat").critical_path_stats() == {"stages": 3,
                                                                        "messages_per_proc": 3}
    assert build_qary_levels(9, 3) == [[(0, 1, 2), (3, 4, 5), (6, 7, 8)], [(0, 3, 6)]]
    assert qary_tree(10, 3).root == 0
    t = parse_tree("levels:[[0,1],[2,3]];[[0,2]]")
    assert t.schedule() == ReductionTree(P=4).schedule()
    for bad in ("binary", "ring:4", "binary:x", "levels:[[0]]"):
        with pytest.raises(TreeError):
            parse_tree(bad)
    with pytest.raises(TreeError):
        ReductionTree(P=4, shape="levels", levels=(((0, 1),),))
    with pytest.raises(TreeError):
        qary_tree(9, 3).device_levels()  # q-ary groups are not pairwise


# ---- core -------------------------------------------------------------------

def test_layouts(golden):
    lay = BlockRowLayout(10, 2, 3)
    assert lay.block_rows == (3, 3, 4) and lay.row_offsets() == [0, 3, 6, 10]
    with pytest.raises(DimensionError):
        BlockRowLayout(5, 3, 2)
    A = np.arange(60.0).reshape(20, 3)
    assert np.array_equal(np.vstack(partition_block_rows(A, 3)), A)
    bc = BlockCyclicLayout(1024, 1024, 128, 2, 4)
    assert np.array_equal(np.array([[bc.owner(i, j) for j in range(8)] for i in range(8)]),
                          golden["misc"]["bc_owner"])
    with pytest.raises(DimensionError):
        BlockCyclicLayout(100, 100, 30, 1, 1)


def test_generators_bit_identical_to_reference(golden):
    g = golden["misc"]
    assert np.array_equal(rng_for(0).standard_normal((1000, 8)), g["normal_s0_1000x8"])
    assert np.array_equal(rng_for(0).uniform(-1, 1, (1000, 8)), g["uniform_s0_1000x8"])
    A = gen_cond_matrix(CondSpec(64, 8, kappa=1e12, seed=3))
    assert np.max(np.abs(A - g["cond_64x8_k1e12_s3"])) <= 1e-15
    with pytest.raises(DimensionError):
        CondSpec(3, 5, kappa=10.0)


# ---- counters -----------------------------------------------------------------

def test_flop_counts_match_reference_model():
    n, m = 16, 3200
    f, d = count_geqr2(m, n)
    model = 2 * m * n ** 2 - (2 / 3) * n ** 3
    assert abs(f - model) <= 0.05 * model and d > 0
    # stacked combine ~ 1/5 of the dense QR of the 2n x n stack (test_householder.py:188-200)
    ratio = count_stacked(80)[0] / count_geqr2(160, 80)[0]
    assert 0.17 <= ratio <= 0.23
    c = FlopCounter()
    c.add_gemm(3, 4, 5)
    assert c.flops == 3 * 5 * 7


def test_comm_recorder():
    rs = [CommRecorder() for _ in range(4)]
    for (lvl, a, b) in oracle.binary_events(4):
        rs[b].record_send(10)
        rs[a].record_recv(10, stage=(lvl, "R"))
    assert critical_path(rs) == (2, 20)


# ---- C-ABI boundary -----------------------------------------------------------

def test_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.LIB_PATH), "build the library first (__graft_entry__.build())"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    header = open(os.path.join(ROOT, "include", "caqr_sm100.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(\w+)\(", header, flags=re.M))
    assert declared == set(_lib.SYMBOLS)
    for s in declared:
        assert hasattr(lib, s), s
    loaded = _lib.load()
    assert loaded.caqr_sm100_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_dropin_package_imports():
    import caqr.caqr
    import caqr.core
    import caqr.householder
    import caqr.trees
    import caqr.tsqr

    assert caqr.trees.ReductionTree is ReductionTree
    assert callable(caqr.tsqr.tsqr_parallel) and callable(caqr.caqr.caqr_factor)
    assert callable(caqr.householder.qr_stacked_triangles)


def test_stream_plan_is_the_binary_tree():
    """Chunk subtrees + upper levels of the streamed TSQR are exactly the
    pairs of the global binary tree (trees.py:52-66), and the chunks tile the
    rows of BlockRowLayout(m, n, P)."""
    from paper_0809_2407_b200.core import BlockRowLayout
    from paper_0809_2407_b200.stream import plan_chunks, upper_events
    from paper_0809_2407_b200.trees import ReductionTree

    for P in [1, 2, 3, 5, 8, 13, 64, 100, 257]:
        m, n = P * 50 + 7, 4
        ref = {(a, b) for grp in ReductionTree(P=P).levels for (a, b) in grp}
        lay = BlockRowLayout(m, n, P)
        for K in [1, 2, 4, 8, 16, 128, 512]:
            got, rows = set(), 0
            for (l0, k, r0, nr) in plan_chunks(m, n, P, K):
                assert r0 == rows == l0 * lay.base
                rows += nr
                assert nr == (k * lay.base if l0 + k < P else m - r0)
                if k > 1:
                    got |= {(l0 + a, l0 + b) for grp in ReductionTree(P=k).levels for (a, b) in grp}
            assert rows == m
            for e in upper_events(P, K):
                got |= {(int(a), int(b)) for a, b, _ in e}
            assert got == ref, (P, K)


def test_split_leaves_wave_fill():
    """Chains per leaf (148 SMs): one chain per SM by default, wave fill for
    the R-only chain kernel."""
    from paper_0809_2407_b200.tsqr import split_leaves

    S = 148
    assert split_leaves(65536, 32, 8, S) == 16                        # C1: 128 chains of 512 rows
    assert split_leaves(1048576, 64, 256, S) == 1                     # C2 (R + Q)
    assert split_leaves(1 << 24, 128, 2048, S, fill=True) == 1        # C3, 1 GPU: 13.8 waves
    assert split_leaves(1 << 22, 128, 512, S, fill=True) == 2         # C3 per GPU at 4 GPUs
    assert split_leaves(1 << 21, 128, 256, S, fill=True) == 4         # C3 per GPU at 8 GPUs
    assert split_leaves(1 << 24, 8, 1024, S) == 1                     # C4 per GPU at 8 GPUs
    assert split_leaves(4096, 64, 1, S) == 8                          # chains stay >= 512 rows
    # n <= 8, R only: more chains than the 148 x 8 warp slots, which the library deals evenly
    assert split_leaves(1 << 24, 8, 1024, S, narrow=True) == 2        # C4 per GPU at 8 GPUs
    assert split_leaves(1 << 27, 8, 8192, S, narrow=True) == 1        # C4, 1 GPU
    assert split_leaves(1 << 20, 8, 64, S, narrow=True) == 32         # 2048 chains of 512 rows
    assert split_leaves(1 << 16, 8, 4, S, narrow=True) == 1           # too short to fill a wave


def test_caqr_grid_layout_needs_a_distributed_job():
    """SPEC caqr_factor(A, layout) with Pr x Pc > 1 runs Algorithm 3 across
    ranks; without a matching torch.distributed job it fails loudly."""
    from paper_0809_2407_b200.caqr import caqr_factor
    from paper_0809_2407_b200.core import BlockCyclicLayout
    from paper_0809_2407_b200.executor import ExecutorError

    A = np.zeros((256, 128))
    with pytest.raises(ExecutorError):
        caqr_factor(A, BlockCyclicLayout(256, 128, 64, 2, 1))


def test_mat1_format_matches_the_reference_layout(tmp_path):
    """MAT1 (matio.py:1-10): 24-byte little-endian header + column-major doubles;
    bad magic / short files raise FormatError; CSV round trip."""
    import struct

    from paper_0809_2407_b200.matio import (FormatError, open_mat1, read_matrix, write_csv,
                                            write_mat1, write_matrix)

    A = np.arange(12, dtype=np.float64).reshape(4, 3) / 7.0
    p = tmp_path / "a.mat"
    write_mat1(p, A)
    raw = p.read_bytes()
    assert raw[:24] == struct.pack("<8sIIII", b"TSQRMAT1", 4, 3, 0, 0)
    assert raw[24:] == A.tobytes(order="F")
    assert np.array_equal(read_matrix(p), A)
    mm = open_mat1(p)
    assert mm.flags.f_contiguous and np.array_equal(np.asarray(mm), A)
    c = tmp_path / "a.csv"
    write_matrix(c, A)
    assert np.array_equal(read_matrix(c), A)
    (tmp_path / "bad.mat").write_bytes(b"NOTAMAT1" + raw[8:])
    with pytest.raises(FormatError):
        read_matrix(tmp_path / "bad.mat")
    (tmp_path / "short.mat").write_bytes(raw[:-8])
    with pytest.raises(FormatError):
        read_matrix(tmp_path / "short.mat")
    B = A.copy()
    B[1, 1] = np.nan
    with pytest.raises(ValueError):
        write_csv(tmp_path / "nan.csv", B)  # as_matrix on write too (matio.py:54-55)
    np.savetxt(tmp_path / "nan.csv", B, delimiter=",")
    with pytest.raises(ValueError):
        read_matrix(tmp_path / "nan.csv")


class _RingSum:
    """SPMD program for LocalExecutor.run: each worker passes its value around
    a ring for P-1 supersteps and sums what it receives."""

    def __init__(self, P):
        self.n_workers = P
        self.n_steps = P

    def setup(self, w):
        return {"acc": float(w), "val": np.array([float(w)])}

    def step(self, w, st, step, inbox):
        from caqr.executor import Message

        for msg in inbox:
            st["acc"] += float(msg.payload[0])
            st["val"] = msg.payload
        if step == self.n_steps - 1:
            return []
        return [Message(w, (w + 1) % self.n_workers, "v", st["val"])]

    def finish(self, w, st):
        return st["acc"]


@pytest.mark.parametrize("threads", [1, 4])
def test_local_executor_runs_reference_programs(threads):
    """caqr.executor keeps the reference API (executor.py:20-94): Message,
    payload_words and LocalExecutor.run -> (results, recorders)."""
    from caqr.executor import ExecutorError, LocalExecutor, Message, payload_words

    assert payload_words(np.zeros((3, 4))) == 12
    assert payload_words({"a": 1.0, "b": (np.zeros(2), None)}) == 3
    assert Message(0, 1, "t", np.zeros(5)).words == 5
    P = 5
    res, recs = LocalExecutor(threads=threads).run(_RingSum(P))
    assert res == [float(P * (P - 1) / 2)] * P
    assert all(r.words_sent == P - 1 and r.words_received == P - 1 for r in recs)

    class Bad(_RingSum):
        def step(self, w, st, step, inbox):
            return [Message((w + 1) % P, w, "x", None)]

    with pytest.raises(ExecutorError):
        LocalExecutor(threads=threads).run(Bad(P))
    with pytest.raises(ValueError):
        LocalExecutor(threads=0)


def test_stacked_flop_count_qary():
    """q-ary stacked profile: reflector j has length 1 + (q-1)(j+1); counts
    equal the reference's own counter (tests/golden/flops_stacked.json,
    oracle/make_golden_flops.py)."""
    import json
    import os

    from paper_0809_2407_b200.counters import count_stacked

    with open(os.path.join(os.path.dirname(__file__), "golden", "flops_stacked.json")) as fh:
        gold = json.load(fh)
    for key, (flops, divs) in gold.items():
        n, q = map(int, key.split("x"))
        assert count_stacked(n, q) == (flops, divs), key


def test_synth_regenerates_reference_bits():
    """paper_0809_2407_b200.synth (the bench's input generator) redraws any row
    range from the recorded Philox states bit for bit like a sequential pass of
    the reference generator (core.rng_for), checked on slices of C3 and C4."""
    from oracle import fullsize
    from paper_0809_2407_b200 import synth

    for cfg, lo, hi in [("c3", 5 * (1 << 20) - 3, 5 * (1 << 20) + 7), ("c4", 2 * (1 << 23) + 11, 2 * (1 << 23) + 40)]:
        got = {}
        synth.chunks(cfg, lo, hi, lambda r0, b: got.__setitem__(r0, b.copy()))
        want = None
        for r0, blk in fullsize.chunks(cfg):
            if r0 + blk.shape[0] > lo:
                if want is None:
                    want = blk[lo - r0:]
                else:
                    want = np.vstack([want, blk])
            if r0 + blk.shape[0] >= hi:
                break
        seq = np.vstack([got[k] for k in sorted(got)])
        assert np.array_equal(seq, want[:hi - lo])


def test_choose_P_sequential_spec_examples():
    """smallest P with mn/P + n(n+1)/2 <= W."""
    from paper_0809_2407_b200.sequential import choose_P_sequential

    assert choose_P_sequential(10 ** 6, 50, 10 ** 6) == 51
    assert choose_P_sequential(100, 5, 10_000) == 1
    with pytest.raises(ValueError, match="too large for fast memory"):
        choose_P_sequential(1000, 50, 1000)


def test_block_store_layout_and_counters(tmp_path):
    """BlockStore on disk: meta.json + A_k.mat in MAT1, counted reads."""
    import json

    from paper_0809_2407_b200.matio import read_mat1
    from paper_0809_2407_b200.sequential import BlockStore

    A = np.random.Generator(np.random.Philox(5)).standard_normal((103, 6))
    st = BlockStore.from_matrix(A, 4, directory=str(tmp_path / "store"))
    meta = json.load(open(tmp_path / "store" / "meta.json"))
    assert meta == {"m": 103, "n": 6, "P": 4, "block_rows": [25, 25, 25, 28]}
    assert np.array_equal(read_mat1(tmp_path / "store" / "A_3.mat"), A[75:])
    again = BlockStore(str(tmp_path / "store"))
    assert np.array_equal(again.read_block(1), A[25:50])
    assert again.counters() == {"blocks_read": 1, "blocks_written": 0, "words_read": 150,
                                "words_written": 0}
