"""GPU parity of the TSQR path (C-ABI kernels) against the CPU oracle.

Tolerances (north star / SURVEY 8(c)):
  R     : max |sn(R_gpu) - sn(R_ref)| <= 1000 eps ||A||_2  (sign-normalised)
  resid : ||A - QR||_F / ||A||_F <= 10 n eps
  orth  : ||Q^T Q - I||_F <= 10 n eps   (chunked-pairwise Gram)
Same-algorithm comparisons (GPU hybrid chain vs oracle hybrid chain) use a
tighter structural tolerance on the implicit-Q factors themselves.
"""

import numpy as np
import pytest
import torch

import oracle
from oracle import EPS

pytestmark = pytest.mark.gpu


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def geom(n):
    from paper_0809_2407_b200 import _lib

    return _lib.geometry(n)


def factor(A, P, want_q=True):
    from paper_0809_2407_b200.tsqr import factor_device

    At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    return factor_device(At, P, want_q=want_q)


@pytest.mark.parametrize("m,n,P", [(600, 8, 1), (1000, 32, 3), (1500, 64, 2), (2000, 128, 2),
                                   (777, 100, 1), (4096, 48, 5), (300, 128, 1)])
def test_leaf_chain_factors_match_oracle(m, n, P):
    """Leaf chain (dense tile + triangle-on-rectangle tiles) and tree factors
    element-wise against the oracle running the same hybrid algorithm."""
    A = philox(m + n).standard_normal((m, n))
    _, h0, ht = geom(n)
    f = factor(A, P)
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    scale = np.linalg.norm(A, 2)
    R = f.R.cpu().numpy()
    assert np.max(np.abs(R - ref["R"])) <= 200 * EPS * scale
    Y = f.Y.cpu().numpy()
    tau = f.tau.cpu().numpy()
    offs = ref["offs"]
    for i, tiles in enumerate(ref["leaves"]):
        b = offs[i + 1] - offs[i]
        bnds = oracle.tsqr.chain_tiles(b, h0, ht)
        Y0, t0 = tiles[0]
        s0, e0 = bnds[0]
        Yg = Y[offs[i] + s0: offs[i] + e0]
        low = np.tril(np.ones_like(Y0, dtype=bool), -1)
        assert np.max(np.abs(Yg[low] - Y0[low])) <= 1e-10, (i, "dense Y")
        assert np.max(np.abs(tau[i, 0] - t0)) <= 1e-12
        for k, ((V, t), (s, e)) in enumerate(zip(tiles[1:], bnds[1:]), start=1):
            Vg = Y[offs[i] + s: offs[i] + e]
            assert np.max(np.abs(Vg - V)) <= 1e-9 * max(1.0, np.max(np.abs(V))), (i, k)
            assert np.max(np.abs(tau[i, k] - t)) <= 1e-12, (i, k)
    if P > 1:
        nY = f.node_Y.cpu().numpy()
        nt = f.node_tau.cpu().numpy()
        for e, (lvl, a, b, Yb, tn) in enumerate(ref["nodes"]):
            assert np.max(np.abs(nY[e] - Yb)) <= 1e-9, e
            assert np.max(np.abs(nt[e] - tn)) <= 1e-12, e


@pytest.mark.parametrize("m,n,P", [(1000, 32, 3), (1500, 64, 2), (2000, 128, 2), (4096, 8, 4),
                                   (999, 17, 3)])
def test_explicit_q_matches_oracle(m, n, P):
    from paper_0809_2407_b200.tsqr import explicit_q_device

    A = philox(7 * m + n).standard_normal((m, n))
    _, h0, ht = geom(n)
    f = factor(A, P)
    Q = explicit_q_device(f).cpu().numpy()
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    Qref = oracle.tsqr_hybrid_q(ref)
    assert np.max(np.abs(Q - Qref)) <= 1e-11
    R = f.R.cpu().numpy()
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS


def test_golden_composed_tsqr(golden):
    """GPU TSQR vs the reference's own composed TSQR (tests/golden/tsqr.npz)."""
    from paper_0809_2407_b200.tsqr import tsqr

    g = golden["tsqr"]
    for tag in sorted({k.rsplit("_", 1)[0] for k in g}):
        A = g[f"{tag}_A"]
        P = int(tag.split("_P")[1])
        n = A.shape[1]
        from paper_0809_2407_b200.trees import ReductionTree

        R, Q = tsqr(A, q="explicit", tree=ReductionTree(P=P))
        assert oracle.r_diff(R, g[f"{tag}_R"]) <= 1000 * EPS, tag
        assert oracle.residual(A, Q, R) <= 10 * n * EPS, tag
        assert oracle.orthogonality(Q) <= 10 * n * EPS, tag
        # Q matches the reference Q column-by-column up to the R sign flips
        # (well-conditioned cases only: for kappa = 1e12 the trailing columns of
        # two backward-stable Q factors legitimately differ by O(eps kappa_j))
        if "1024x64" in tag:
            continue
        d = np.sign(np.diag(R)) * np.sign(np.diag(g[f"{tag}_R"]))
        assert np.max(np.abs(Q * d - g[f"{tag}_Q"])) <= 1e-6, tag


def test_known_answers():
    from paper_0809_2407_b200.tsqr import tsqr

    # identity stack -> R = I (up to signs), Q has a single +-1 per column
    A = np.vstack([np.eye(8)] * 64)
    R, Q = tsqr(A, leaf_rows=64, q="explicit")
    assert np.allclose(np.abs(R), np.sqrt(64) * np.eye(8), atol=1e-13)
    # [I; 0] -> R = I bitwise, Q = [I; 0] (test_householder.py:160-163, 299-302)
    A = np.zeros((512, 16))
    A[:16] = np.eye(16)
    R, Q = tsqr(A, leaf_rows=128, q="explicit")
    assert np.array_equal(R, np.eye(16))
    assert np.array_equal(Q, A)
    # zero matrix: R = 0, Q = [I; 0] (tau = 0 everywhere)
    R, Q = tsqr(np.zeros((1024, 32)), leaf_rows=256, q="explicit")
    assert np.array_equal(R, np.zeros((32, 32)))
    E = np.zeros((1024, 32))
    E[:32] = np.eye(32)
    assert np.array_equal(Q, E)
    # positive upper-triangular block on top of zeros: unchanged, bitwise
    T = np.triu(philox(3).standard_normal((24, 24)))
    np.fill_diagonal(T, np.abs(np.diag(T)) + 1.0)
    A = np.zeros((800, 24))
    A[:24] = T
    R, _ = tsqr(A, leaf_rows=400, q="implicit")  # dense first tile = qr_unblocked: tau = 0
    assert np.array_equal(R, T)
    # R only: every leaf chain starts from R = 0 (CAQR_TUNE_ZSTART), so the
    # first reflector of each column flips its row -- the same R up to signs
    R = tsqr(A, leaf_rows=400)
    assert np.array_equal(np.abs(R), np.abs(T)) or oracle.r_diff(R, T) <= 10 * EPS


def test_rejects_bad_input():
    from paper_0809_2407_b200.core import DimensionError
    from paper_0809_2407_b200.tsqr import tsqr

    with pytest.raises(DimensionError):
        tsqr(np.ones((4, 8)))
    with pytest.raises(DimensionError):
        tsqr(np.ones(8))
    with pytest.raises(DimensionError):
        tsqr(np.ones((4096, 129)))
    A = philox(1).standard_normal((1000, 16))
    A[517, 3] = np.nan
    with pytest.raises(ValueError):
        tsqr(A, leaf_rows=250)
    A[517, 3] = np.inf
    with pytest.raises(ValueError):
        tsqr(A, leaf_rows=250)


def test_apply_q_round_trips():
    from paper_0809_2407_b200.tsqr import apply_q_device

    m, n = 5000, 40
    A = philox(11).standard_normal((m, n))
    _, h0, ht = geom(n)
    f = factor(A, 4)
    ref = oracle.tsqr_hybrid(A, 4, h0, ht)
    C = philox(12).standard_normal((m, 5))
    Ct = torch.from_numpy(C).cuda()
    QtC = apply_q_device(f, Ct, transpose=True).cpu().numpy()
    assert np.max(np.abs(QtC - oracle.tsqr.tsqr_hybrid_apply(ref, C, True))) <= 1e-11
    back = apply_q_device(f, torch.from_numpy(QtC).cuda(), transpose=False).cpu().numpy()
    assert np.max(np.abs(back - C)) <= 100 * n * EPS * np.linalg.norm(C)
    # thin apply: Q (R x) == A x
    x = philox(13).standard_normal((n, 3))
    Rx = torch.from_numpy(f.R.cpu().numpy() @ x).cuda()
    Ax = apply_q_device(f, Rx, transpose=False).cpu().numpy()
    assert np.max(np.abs(Ax - A @ x)) <= 100 * n * EPS * np.linalg.norm(A) * np.linalg.norm(x)


def test_tsqr_parallel_spec_api():
    from paper_0809_2407_b200 import DeviceExecutor, partition_block_rows
    from paper_0809_2407_b200.counters import FlopCounter
    from paper_0809_2407_b200.tsqr import tsqr_explicit_q, tsqr_parallel

    A = philox(21).standard_normal((4096, 16))
    ex = DeviceExecutor(record=True)
    c = FlopCounter()
    f = tsqr_parallel(ex, partition_block_rows(A, 8), counter=c)
    Q = tsqr_explicit_q(f)
    assert isinstance(Q, np.ndarray)
    R = f.R_out()
    assert oracle.residual(A, Q, R) <= 10 * 16 * EPS
    # census: log2(P) messages of n(n+1)/2 words on the critical path
    from paper_0809_2407_b200.counters import critical_path

    msgs, words = critical_path(ex.recorders)
    assert msgs == 3 and words == 3 * 16 * 17 // 2
    model = 2 * 4096 * 16 ** 2 - (2 / 3) * 16 ** 3
    assert abs(c.flops - model) <= 0.05 * model


def test_c1_full_size():
    """Config 1: 65536 x 32 N(0,1), 8 leaves of 8192, R + explicit Q."""
    from paper_0809_2407_b200.tsqr import tsqr

    A = philox(0).standard_normal((65536, 32))
    R, Q = tsqr(A, leaf_rows=8192, q="explicit")
    ref = oracle.tsqr_reference(A, 8)
    n = 32
    assert oracle.r_diff(R, ref["R"]) <= 1000 * EPS
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS


@pytest.mark.parametrize("m,n,P", [(16384 * 3 + 77, 8, 3), (5000, 5, 2), (1 << 16, 8, 4), (999, 1, 3),
                                   (40000, 7, 1)])
def test_narrow_r_only_matches_oracle(m, n, P):
    """n <= 8, R only: lane-private chains + in-warp tree (k_leaf_narrow)."""
    from paper_0809_2407_b200.tsqr import tsqr
    from paper_0809_2407_b200.trees import ReductionTree

    A = philox(m + n).uniform(-1, 1, (m, n))
    R = tsqr(A, tree=ReductionTree(P=P))
    Rref = oracle.tsqr_reference(A, P)["R"]
    assert oracle.r_diff(R, Rref) <= 1000 * EPS
    # ill-conditioned, same path
    from paper_0809_2407_b200.core import CondSpec, gen_cond_matrix

    A = gen_cond_matrix(CondSpec(4096, n, kappa=1e12, seed=n))
    R = tsqr(A, leaf_rows=1024)
    Rref = np.linalg.qr(A, mode="r")
    assert oracle.r_diff(R, Rref) <= 1000 * EPS


def test_narrow_rejects_nonfinite():
    from paper_0809_2407_b200.tsqr import tsqr

    A = philox(5).standard_normal((20000, 8))
    A[12345, 7] = np.inf
    with pytest.raises(ValueError):
        tsqr(A, leaf_rows=4096)


@pytest.mark.parametrize("m,n,leaf,K", [(100037, 128, 4096, 4), (65536 + 999, 64, 2048, 2),
                                        (1 << 20, 8, 16384, 8), (50000, 32, 1000, 16)])
def test_streamed_r_is_bitwise_the_device_r(m, n, leaf, K):
    """Host-resident A streamed in chunks of K leaves (paper_0809_2407_b200.stream)
    gives the device-resident path's R bit for bit (same leaves, same tree)."""
    from paper_0809_2407_b200.stream import tsqr_stream
    from paper_0809_2407_b200.tsqr import _leaves_for, factor_device, split_leaves, tsqr

    A = philox(m + n).standard_normal((m, n))
    P = _leaves_for(m, n, leaf)
    P *= split_leaves(m, n, P, fill=n > 8)
    Rdev = factor_device(torch.from_numpy(A).cuda(), P).R.cpu().numpy()
    Rs = tsqr_stream(A, P, chunk_leaves=K).cpu().numpy()  # pageable: staged
    assert np.array_equal(Rs, Rdev)
    Ap = torch.from_numpy(A).pin_memory()
    assert np.array_equal(tsqr_stream(Ap, P, chunk_leaves=K, buffers=2).cpu().numpy(), Rdev)
    # the public entry point streams host input by default
    assert np.array_equal(tsqr(A, leaf_rows=leaf), Rdev)
    assert oracle.r_diff(Rdev, np.linalg.qr(A, mode="r")) <= 1000 * EPS


def test_streamed_rejects_nonfinite():
    from paper_0809_2407_b200.tsqr import tsqr

    A = philox(5).standard_normal((40000, 16))
    A[33333, 3] = np.inf
    with pytest.raises(ValueError):
        tsqr(A, leaf_rows=1000)


def test_tuning_variants_keep_parity():
    """The supported tuning knobs (CAQR_TUNE_CHAIN_HT_128 = 24, CAQR_TUNE_ZSTART
    = 0) change the tiling / first tile only: parity holds for each."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import tsqr

    A = philox(31).standard_normal((20000, 100))
    Rref = np.linalg.qr(A, mode="r")
    scale = np.linalg.norm(A, 2)
    try:
        _lib.tune(_lib.TUNE_CHAIN_HT[128], 24)
        R, Q = tsqr(A, leaf_rows=5000, q="explicit")
        assert oracle.r_diff(R, Rref, scale) <= 1000 * EPS
        assert oracle.orthogonality(Q) <= 10 * 100 * EPS
        assert oracle.residual(A, Q, R) <= 10 * 100 * EPS
    finally:
        _lib.reset_tuning()
    try:
        _lib.tune(_lib.TUNE_ZSTART, 0)
        R0 = tsqr(A, leaf_rows=5000)  # dense first tile, ring tree
        assert oracle.r_diff(R0, Rref, scale) <= 1000 * EPS
    finally:
        _lib.reset_tuning()
    assert oracle.r_diff(tsqr(A, leaf_rows=5000), Rref, scale) <= 1000 * EPS


@pytest.mark.parametrize("m,n,leaf,K", [(70001, 128, 4096, 2), (200000, 8, 16384, 4), (30000, 50, 1000, 8)])
def test_tsqr_from_mat1_file_is_bitwise_the_in_memory_r(tmp_path, m, n, leaf, K):
    """TSQR streamed from a column-major MAT1 file (transpose on the GPU) gives
    tsqr()'s R bit for bit; also through the chunked path with K leaves per chunk."""
    from paper_0809_2407_b200.matio import open_mat1, tsqr_mat1, write_mat1
    from paper_0809_2407_b200.stream import tsqr_stream
    from paper_0809_2407_b200.tsqr import _leaves_for, factor_device, split_leaves, tsqr

    A = philox(m * 3 + n).standard_normal((m, n))
    p = tmp_path / "a.mat"
    write_mat1(p, A)
    R = tsqr(A, leaf_rows=leaf)
    assert np.array_equal(tsqr_mat1(p, leaf_rows=leaf), R)
    P = _leaves_for(m, n, leaf)
    P *= split_leaves(m, n, P, fill=n > 8)
    Rk = tsqr_stream(open_mat1(p), P, chunk_leaves=K).cpu().numpy()
    assert np.array_equal(Rk, factor_device(torch.from_numpy(A).cuda(), P).R.cpu().numpy())


@pytest.mark.parametrize("v16", [True, False])
def test_dmma_ring_leaf_parity(v16):
    """CAQR_TUNE_DMMA = 1 (default): R-only leaves with n in (64, 128] on the
    DMMA warp ring (16-row register tiles, 8-column Level-2 panels with
    look-ahead, compact-WY updates and T on the FP64 tensor cores).  R against
    LAPACK, sign-normalised; odd n / lda take the 8-byte cp.async staging path."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    shapes = [(4096, 128, 2), (20000, 100, 4), (3000, 72, 1), (9001, 128, 3), (1 << 16, 128, 4)]
    if not v16:
        shapes = [(5000, 99, 2), (4099, 127, 3)]
    try:
        _lib.tune(_lib.TUNE_DMMA, 1)
        for (m, n, P) in shapes:
            A = philox(m + n).standard_normal((m, n))
            R = factor_device(torch.from_numpy(A).cuda(), P).R.cpu().numpy()
            assert np.array_equal(R, np.triu(R))
            d = oracle.r_diff(R, np.linalg.qr(A, mode="r"), np.linalg.norm(A, 2))
            assert d <= 1000 * EPS, (m, n, P, d / EPS)
        # rank-deficient and zero columns (sigma = 0 / tau = 0 reflectors inside a
        # panel): R is no longer unique, so check R^T R = A^T A instead
        A = philox(3).standard_normal((4096, 96))
        A[:, 10] = 0.0
        A[:, 40] = A[:, 41]
        R = factor_device(torch.from_numpy(A).cuda(), 2).R.cpu().numpy()
        assert np.linalg.norm(R.T @ R - A.T @ A) <= 1000 * EPS * np.linalg.norm(A, 2) ** 2
        A = philox(7).standard_normal((5000, 96))
        A[4321, 50] = np.nan
        with pytest.raises(ValueError):
            factor_device(torch.from_numpy(A).cuda(), 2)
    finally:
        _lib.reset_tuning()


def test_dmma_ring_matches_rank1_ring():
    """The DMMA ring and the rank-1 ring (CAQR_TUNE_DMMA = 0) give the same R up
    to row signs on a C3-shaped slice (32 leaves of 8192 x 128)."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    A = torch.from_numpy(philox(11).standard_normal((32 * 8192, 128))).cuda()
    Rd = factor_device(A, 32).R.cpu().numpy()
    try:
        _lib.tune(_lib.TUNE_DMMA, 0)
        Rr = factor_device(A, 32).R.cpu().numpy()
    finally:
        _lib.reset_tuning()
    nA = np.linalg.norm(Rr, 2)
    assert oracle.r_diff(Rd, Rr, nA) <= 1000 * EPS


@pytest.mark.parametrize("shape", [(8 * 2048, 128, 8, 300), (3 * 1500 + 77, 100, 3, 129),
                                   (4096, 128, 2, 64), (8 * 2048, 128, 8, 37 * 128 + 5)])
def test_dmma_leaf_apply_matches_ring(shape):
    """CAQR_TUNE_DMMA_APPLY = 1 (default): Q^T C of n in (64, 128] chain leaves
    on the DMMA ring (compact WY per 8-reflector panel, T from the Neumann
    product; 32-column CTAs when the launch is small, 128-column CTAs for the
    last shape) and the DMMA tree apply equal the reflector rings (= 0), and
    Q (Q^T C) = C."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, factor_device

    m, n, P, k = shape
    A = torch.from_numpy(philox(m + k).standard_normal((m, n))).cuda()
    C = torch.from_numpy(philox(m - k).standard_normal((m, k))).cuda()
    f = factor_device(A, P, want_q=True)
    Qd = apply_q_device(f, C, transpose=True)
    try:
        _lib.tune(_lib.TUNE_DMMA_APPLY, 0)
        Qr = apply_q_device(f, C, transpose=True)
    finally:
        _lib.reset_tuning()
    scale = torch.linalg.norm(C).item()
    assert torch.linalg.norm(Qd - Qr).item() <= 100 * n * EPS * scale
    # round trip: Q (Q^T C) = C
    back = apply_q_device(f, Qd, transpose=False)
    assert torch.linalg.norm(back - C).item() <= 100 * n * EPS * scale


def test_dmma_kernels_random_shapes():
    """Randomised cross-check (tools/stress_dmma.py, 10 shapes): DMMA leaf factor
    (R only and Q-keeping), DMMA leaf apply and tree apply vs the rank-1 /
    reflector rings, n in (64, 128], ragged leaves, narrow and wide column counts."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, factor_device

    rng = np.random.default_rng(77)

    def sgn(R):
        return R * torch.sign(torch.diagonal(R)).unsqueeze(1)

    for _ in range(10):
        n = int(rng.integers(65, 129))
        P = int(rng.integers(1, 9))
        m = P * int(rng.integers(max(n, 300), 2500)) + int(rng.integers(0, 50))
        k = int(rng.choice([int(rng.integers(1, 200)), int(rng.integers(2000, 5000))]))
        A = torch.from_numpy(rng.standard_normal((m, n))).cuda()
        C = torch.from_numpy(rng.standard_normal((m, k))).cuda()
        f = factor_device(A, P, want_q=True)
        R1 = factor_device(A, P).R
        Qd = apply_q_device(f, C, transpose=True)
        try:
            _lib.tune(_lib.TUNE_DMMA, 0)
            _lib.tune(_lib.TUNE_DMMA_APPLY, 0)
            f0 = factor_device(A, P, want_q=True)
            R0 = factor_device(A, P).R
            Qr = apply_q_device(f0, C, transpose=True)
        finally:
            _lib.reset_tuning()
        nA = torch.linalg.norm(A, 2).item()
        assert (sgn(R1) - sgn(R0)).abs().max().item() <= 100 * EPS * nA, (m, n, P)
        assert (f.R - f0.R).abs().max().item() <= 100 * EPS * nA, (m, n, P)
        assert torch.linalg.norm(Qd - Qr).item() <= 100 * EPS * torch.linalg.norm(C).item(), (m, n, P, k)


@pytest.mark.parametrize("m,n,P", [(1500, 64, 2), (4096, 48, 5), (999, 33, 3), (20000, 64, 4)])
def test_dmma_ring_np64_matches_oracle(m, n, P):
    """CAQR_TUNE_DMMA = 2 with CAQR_TUNE_CHAIN_HT_64 = 16: leaves with n in (32, 64] on
    the NP = 64 DMMA ring (two CTAs per SM).  Its chain-tile factors (Y, tau) and the
    tree factors against the oracle's hybrid chain element-wise, explicit Q against the
    oracle's Q, and the R-only (zero-start) leaves against LAPACK; odd n takes the 8-byte
    staging path."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

    A = philox(5 * m + n).standard_normal((m, n))
    try:
        _lib.tune(_lib.TUNE_DMMA, 2)
        _lib.tune(_lib.TUNE_CHAIN_HT[64], 16)
        _, h0, ht = geom(n)
        assert ht == 16
        f = factor(A, P)
        Q = explicit_q_device(f).cpu().numpy()
        Rz = factor(A, P, want_q=False).R.cpu().numpy()
    finally:
        _lib.reset_tuning()
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    scale = np.linalg.norm(A, 2)
    R = f.R.cpu().numpy()
    assert np.max(np.abs(R - ref["R"])) <= 200 * EPS * scale
    Y, tau, offs = f.Y.cpu().numpy(), f.tau.cpu().numpy(), ref["offs"]
    for i, tiles in enumerate(ref["leaves"]):
        bnds = oracle.tsqr.chain_tiles(offs[i + 1] - offs[i], h0, ht)
        for k, ((V, t), (s, e)) in enumerate(zip(tiles[1:], bnds[1:]), start=1):
            Vg = Y[offs[i] + s: offs[i] + e]
            assert np.max(np.abs(Vg - V)) <= 1e-9 * max(1.0, np.max(np.abs(V))), (i, k)
            assert np.max(np.abs(tau[i, k] - t)) <= 1e-12, (i, k)
    Qref = oracle.tsqr_hybrid_q(ref)
    assert np.max(np.abs(Q - Qref)) <= 1e-11
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    assert np.array_equal(Rz, np.triu(Rz))
    assert oracle.r_diff(Rz, np.linalg.qr(A, mode="r"), scale) <= 1000 * EPS


@pytest.mark.parametrize("n,variant", [(64, 1), (64, 2), (64, 3), (40, 1), (128, 1), (99, 1)])
def test_dmma_leaf_q_matches_ring(n, variant):
    """CAQR_TUNE_DMMA_Q (1 = NP 64 with 64-column CTAs, 2 = 32-column CTAs, 3 = one CTA per
    SM): Q C on the backward DMMA ring + reverse-panel dense tile equals the
    reflector-by-reflector ring (= 0) for explicit Q, thin Q C (S path, zero-initialised
    rows) and full Q C (C's own rows), and Q^T (Q C) = C."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device, factor_device

    m, P, k = 3 * 2500 + 37, 3, 300
    A = torch.from_numpy(philox(n + variant).standard_normal((m, n))).cuda()
    Cf = torch.from_numpy(philox(2 * n).standard_normal((m, k))).cuda()
    Ct = torch.from_numpy(philox(3 * n).standard_normal((n, k))).cuda()
    try:
        _lib.tune(_lib.TUNE_DMMA, 2)
        _lib.tune(_lib.TUNE_CHAIN_HT[64], 16)
        f = factor_device(A, P, want_q=True)
        out = []
        for qv in (variant, 0):
            _lib.tune(_lib.TUNE_DMMA_Q, qv)
            out.append((explicit_q_device(f), apply_q_device(f, Ct, transpose=False),
                        apply_q_device(f, Cf, transpose=False)))
        back = apply_q_device(f, out[0][2], transpose=True)  # same chain geometry as f
    finally:
        _lib.reset_tuning()
    (Qd, Td, Fd), (Qr, Tr, Fr) = out
    assert (Qd - Qr).abs().max().item() <= 1e-12
    assert torch.linalg.norm(Td - Tr).item() <= 100 * n * EPS * torch.linalg.norm(Ct).item()
    assert torch.linalg.norm(Fd - Fr).item() <= 100 * n * EPS * torch.linalg.norm(Cf).item()
    assert torch.linalg.norm(back - Cf).item() <= 100 * n * EPS * torch.linalg.norm(Cf).item()


@pytest.mark.parametrize("dmma,ht", [(1, 24), (1, 16), (0, 24)])
def test_np64_chain_variants_keep_parity(dmma, ht):
    """n in (32, 64] off the default DMMA path: the rank-1 chain with 24- or 16-row
    tiles (CAQR_TUNE_DMMA = 1 / 0, CAQR_TUNE_CHAIN_HT_64) and the reflector-ring Q / Q^T
    applies; R, explicit Q and Q^T C against LAPACK / the oracle's invariants."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device, factor_device

    m, n, P = 6000, 56, 3
    A = philox(4 * ht + dmma).standard_normal((m, n))
    C = torch.from_numpy(philox(9).standard_normal((m, 70))).cuda()
    try:
        _lib.tune(_lib.TUNE_DMMA, dmma)
        _lib.tune(_lib.TUNE_CHAIN_HT[64], ht)
        assert geom(n)[2] == ht
        f = factor(A, P)
        Q = explicit_q_device(f).cpu().numpy()
        QtC = apply_q_device(f, C, transpose=True)
        back = apply_q_device(f, QtC, transpose=False)
        Rz = factor(A, P, want_q=False).R.cpu().numpy()
    finally:
        _lib.reset_tuning()
    R = f.R.cpu().numpy()
    scale = np.linalg.norm(A, 2)
    assert oracle.r_diff(R, np.linalg.qr(A, mode="r"), scale) <= 1000 * EPS
    assert oracle.r_diff(Rz, np.linalg.qr(A, mode="r"), scale) <= 1000 * EPS
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    assert torch.linalg.norm(back - C).item() <= 100 * n * EPS * torch.linalg.norm(C).item()


@pytest.mark.parametrize("n,variant", [(64, 1), (64, 2), (64, 3), (37, 1)])
def test_dmma_leaf_qt_np64_matches_ring(n, variant):
    """CAQR_TUNE_DMMA_APPLY for n in (32, 64] (k_leaf_q_dmma with TR: dense tile forward,
    then the chain ring forward, T^T): Q^T C equals the reflector ring (= 0), on ragged
    leaves and a column count that is not a multiple of the CTA width, and Q (Q^T C) = C."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, factor_device

    m, P, k = 4 * 1900 + 13, 4, 150
    A = torch.from_numpy(philox(7 * n + variant).standard_normal((m, n))).cuda()
    C = torch.from_numpy(philox(8 * n).standard_normal((m, k))).cuda()
    f = factor_device(A, P, want_q=True)
    try:
        _lib.tune(_lib.TUNE_DMMA_APPLY, variant)
        Qd = apply_q_device(f, C, transpose=True)
        back = apply_q_device(f, Qd, transpose=False)
        _lib.tune(_lib.TUNE_DMMA_APPLY, 0)
        Qr = apply_q_device(f, C, transpose=True)
    finally:
        _lib.reset_tuning()
    scale = torch.linalg.norm(C).item()
    assert torch.linalg.norm(Qd - Qr).item() <= 100 * n * EPS * scale
    assert torch.linalg.norm(back - C).item() <= 100 * n * EPS * scale


@pytest.mark.parametrize("n", [64, 40, 128, 100])
def test_dmma_tree_apply_matches_ring(n):
    """CAQR_TUNE_DMMA_TREE = 1 (default): the tree-level Q / Q^T (STACKED node factors,
    k_tree_apply_dmma, both directions, zero partner blocks for explicit Q / thin Q C) equals
    the reflector-by-reflector k_tree_apply (= 0)."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device, factor_device

    m, P, k = 8 * 700 + 5, 8, 90
    A = torch.from_numpy(philox(11 * n).standard_normal((m, n))).cuda()
    Cf = torch.from_numpy(philox(12 * n).standard_normal((m, k))).cuda()
    Ct = torch.from_numpy(philox(13 * n).standard_normal((n, k))).cuda()
    f = factor_device(A, P, want_q=True)
    out = []
    try:
        for tv in (1, 0):
            _lib.tune(_lib.TUNE_DMMA_TREE, tv)
            out.append((explicit_q_device(f), apply_q_device(f, Ct, transpose=False),
                        apply_q_device(f, Cf, transpose=False), apply_q_device(f, Cf, transpose=True)))
    finally:
        _lib.reset_tuning()
    for d, r, C in zip(out[0], out[1], (None, Ct, Cf, Cf)):
        scale = 1.0 if C is None else torch.linalg.norm(C).item()
        assert torch.linalg.norm(d - r).item() <= 100 * n * EPS * max(scale, np.sqrt(n))


@pytest.mark.parametrize("n", [32, 20])
def test_dmma_np32_variants_match_ring(n):
    """The DMMA paths for n <= 32 (k_tree_apply_dmma and k_leaf_q_dmma<32>, defaults;
    tuning values 2 / 4 / 4 select the same kernels) equal the reflector rings
    (k_tree_apply_w32, k_leaf_apply; all three keys = 0) for explicit Q, thin and full Q C,
    and Q^T C."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import apply_q_device, explicit_q_device, factor_device

    m, P, k = 4 * 1200 + 9, 4, 45
    A = torch.from_numpy(philox(21 * n).standard_normal((m, n))).cuda()
    Cf = torch.from_numpy(philox(22 * n).standard_normal((m, k))).cuda()
    Ct = torch.from_numpy(philox(23 * n).standard_normal((n, k))).cuda()
    f = factor_device(A, P, want_q=True)
    out = []
    try:
        for tv in ((2, 4, 4), (0, 0, 0)):
            _lib.tune(_lib.TUNE_DMMA_TREE, tv[0])
            _lib.tune(_lib.TUNE_DMMA_Q, tv[1])
            _lib.tune(_lib.TUNE_DMMA_APPLY, tv[2])
            out.append((explicit_q_device(f), apply_q_device(f, Ct, transpose=False),
                        apply_q_device(f, Cf, transpose=False), apply_q_device(f, Cf, transpose=True)))
    finally:
        _lib.reset_tuning()
    for d, r, C in zip(out[0], out[1], (None, Ct, Cf, Cf)):
        scale = 1.0 if C is None else torch.linalg.norm(C).item()
        assert torch.linalg.norm(d - r).item() <= 100 * n * EPS * max(scale, np.sqrt(n))


@pytest.mark.parametrize("n", [8, 17, 32, 40, 64])
def test_dmma_tree_factor_matches_cta_factor(n):
    """CAQR_TUNE_DMMA_TREE_FACTOR = 1 (default, n <= 64): the STACKED node factors
    (k_tree_factor_dmma: column-block warps, Level-2 panels, compact-WY updates) equal
    k_tree_factor / k_tree_factor_w32 (= 0) in node Y, tau and R, every node reflector is
    orthogonal to rounding (tau (1 + |y|^2) = 2), and explicit Q meets the north-star
    bounds."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import explicit_q_device, factor_device

    m, P = 8 * 600 + 3, 8
    A = philox(31 * n).standard_normal((m, n))
    At = torch.from_numpy(A).cuda()
    f1 = factor_device(At, P, want_q=True)
    Q1 = explicit_q_device(f1).cpu().numpy()
    try:
        _lib.tune(_lib.TUNE_DMMA_TREE_FACTOR, 0)
        f0 = factor_device(At, P, want_q=True)
    finally:
        _lib.reset_tuning()
    scale = np.linalg.norm(A, 2)
    assert (f1.R - f0.R).abs().max().item() <= 100 * EPS * scale
    assert (f1.node_Y - f0.node_Y).abs().max().item() <= 1e-13
    assert (f1.node_tau - f0.node_tau).abs().max().item() <= 1e-14
    Y, tau = f1.node_Y.cpu().numpy(), f1.node_tau.cpu().numpy()
    for e in range(Y.shape[0]):
        for j in range(n):
            if tau[e, j]:
                assert abs(tau[e, j] * (1 + Y[e, :, j] @ Y[e, :, j]) - 2) <= 8 * EPS, (e, j)
    R = f1.R.cpu().numpy()
    assert oracle.residual(A, Q1, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q1) <= 10 * n * EPS


@pytest.mark.parametrize("m,n,P", [(1500, 32, 2), (4096, 20, 5), (999, 9, 3)])
def test_dmma_ring_np32_matches_oracle(m, n, P):
    """CAQR_TUNE_DMMA = 3 (opt-in): leaves with n <= 32 on the NP = 32 DMMA ring; chain-tile
    factors (Y, tau) against the oracle's hybrid chain, explicit Q against the oracle's Q, and
    R-only (zero-start) leaves against LAPACK."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import explicit_q_device

    A = philox(9 * m + n).standard_normal((m, n))
    try:
        _lib.tune(_lib.TUNE_DMMA, 3)
        _, h0, ht = geom(n)
        f = factor(A, P)
        Q = explicit_q_device(f).cpu().numpy()
        _lib.tune(_lib.TUNE_NARROW, 0)  # n = 9 would take the lane-private kernel otherwise
        Rz = factor(A, P, want_q=False).R.cpu().numpy()
    finally:
        _lib.reset_tuning()
    ref = oracle.tsqr_hybrid(A, P, h0, ht)
    scale = np.linalg.norm(A, 2)
    R = f.R.cpu().numpy()
    assert np.max(np.abs(R - ref["R"])) <= 200 * EPS * scale
    Y, tau, offs = f.Y.cpu().numpy(), f.tau.cpu().numpy(), ref["offs"]
    for i, tiles in enumerate(ref["leaves"]):
        bnds = oracle.tsqr.chain_tiles(offs[i + 1] - offs[i], h0, ht)
        for k, ((V, t), (s, e)) in enumerate(zip(tiles[1:], bnds[1:]), start=1):
            Vg = Y[offs[i] + s: offs[i] + e]
            assert np.max(np.abs(Vg - V)) <= 1e-9 * max(1.0, np.max(np.abs(V))), (i, k)
            assert np.max(np.abs(tau[i, k] - t)) <= 1e-12, (i, k)
    assert np.max(np.abs(Q - oracle.tsqr_hybrid_q(ref))) <= 1e-11
    assert oracle.residual(A, Q, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q) <= 10 * n * EPS
    assert oracle.r_diff(Rz, np.linalg.qr(A, mode="r"), scale) <= 1000 * EPS


@pytest.mark.parametrize("m,n,P", [(300, 32, 2), (5000, 20, 3), (2000, 64, 4), (129, 64, 1),
                                   (4100, 8, 2)])
def test_dmma_dense_tile_matches_cta_sweep(m, n, P):
    """CAQR_TUNE_DMMA_DENSE = 1 (opt-in, n <= 64): the dense first tile on
    k_leaf_dense_dmma equals the CTA sweep k_leaf_dense (default) in Y (LAPACK layout), tau
    and R, including leaves shorter than the tile; explicit Q meets the north-star bounds."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import explicit_q_device

    A = philox(13 * m + n).standard_normal((m, n))
    f0 = factor(A, P)
    try:
        _lib.tune(_lib.TUNE_DMMA_DENSE, 1)
        f1 = factor(A, P)
        Q1 = explicit_q_device(f1).cpu().numpy()
    finally:
        _lib.reset_tuning()
    scale = np.linalg.norm(A, 2)
    assert (f1.R - f0.R).abs().max().item() <= 100 * EPS * scale
    assert (f1.Y - f0.Y).abs().max().item() <= 1e-12 * max(1.0, f0.Y.abs().max().item())
    assert (f1.tau - f0.tau).abs().max().item() <= 1e-13
    R = f1.R.cpu().numpy()
    assert oracle.residual(A, Q1, R) <= 10 * n * EPS
    assert oracle.orthogonality(Q1) <= 10 * n * EPS


@pytest.mark.parametrize("cc", [4, 3, 2])
def test_split_role_leaves_bitwise_equal_to_ring(cc):
    """CAQR_TUNE_CC = 4 / 3 (default 4): the split-role ring with 16 / 12 tiles in
    tensor memory; 2: with 8 tiles in shared memory.  All run the DMMA warp
    ring's arithmetic (generation warps + update warps): R bitwise equal to
    CAQR_TUNE_CC = 0, and within the R bar of LAPACK.  Shapes cover ragged
    leaves, n < 128 (dead padded blocks), more and fewer tiles than slots."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    try:
        for (m, n, P) in [(4096, 128, 2), (20000, 100, 4), (3000, 72, 1), (9001, 128, 3),
                          (148 * 512 + 77, 120, 148), (100, 65, 1)]:
            A = torch.from_numpy(philox(m + 7 * n).standard_normal((m, n))).cuda()
            _lib.tune(_lib.TUNE_CC, cc)
            Rc = factor_device(A, P).R.cpu().numpy()
            _lib.tune(_lib.TUNE_CC, 0)
            R0 = factor_device(A, P).R.cpu().numpy()
            assert np.array_equal(Rc, R0)
            assert oracle.r_diff(Rc, np.linalg.qr(A.cpu().numpy(), mode="r"),
                                 np.linalg.norm(A.cpu().numpy(), 2)) <= 1000 * EPS
        A = philox(7).standard_normal((5000, 96))
        A[4321, 50] = np.nan
        _lib.tune(_lib.TUNE_CC, cc)
        with pytest.raises(ValueError):
            factor_device(torch.from_numpy(A).cuda(), 2)
    finally:
        _lib.reset_tuning()


@pytest.mark.parametrize("cc", [5, 6])
def test_tall_tile_leaves_match_ring_and_lapack(cc):
    """CAQR_TUNE_CC = 5 (default) / 6: the split-role ring with 4 tiles of 64 rows /
    8 tiles of 32 rows in tensor memory (k_leaf_tt).  Same Householder chain with
    taller rectangles per step (qr_triangle_on_rect, householder.py:297-332), so R
    agrees with the 16-row ring to rounding (not bitwise) and with LAPACK within the
    R bar; run-to-run bitwise.  Shapes cover ragged leaves and last tiles, n < 128,
    more and fewer tiles than slots, an ill-conditioned input and the NaN flag."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    try:
        for (m, n, P) in [(4096, 128, 2), (20000, 100, 4), (3000, 72, 1), (9001, 128, 3),
                          (148 * 512 + 77, 120, 148), (100, 65, 1), (129, 128, 1), (200, 128, 1)]:
            A = torch.from_numpy(philox(m + 7 * n).standard_normal((m, n))).cuda()
            _lib.tune(_lib.TUNE_CC, cc)
            Rc = factor_device(A, P).R.cpu().numpy()
            assert np.array_equal(Rc, factor_device(A, P).R.cpu().numpy())
            _lib.tune(_lib.TUNE_CC, 0)
            R0 = factor_device(A, P).R.cpu().numpy()
            nrm = np.linalg.norm(A.cpu().numpy(), 2)
            assert oracle.r_diff(Rc, R0, nrm) <= 50 * EPS
            assert oracle.r_diff(Rc, np.linalg.qr(A.cpu().numpy(), mode="r"), nrm) <= 1000 * EPS
        # kappa = 1e10: R^T R = A^T A to working accuracy (backward stability of the chain)
        rng = philox(99)
        U, _ = np.linalg.qr(rng.standard_normal((6000, 96)))
        V, _ = np.linalg.qr(rng.standard_normal((96, 96)))
        A = (U * np.logspace(0, -10, 96)) @ V.T
        _lib.tune(_lib.TUNE_CC, cc)
        R = factor_device(torch.from_numpy(A).cuda(), 3).R.cpu().numpy()
        assert np.linalg.norm(R.T @ R - A.T @ A) <= 100 * 96 * EPS * np.linalg.norm(A, 2) ** 2
        A = philox(7).standard_normal((5000, 96))
        A[4321, 50] = np.nan
        with pytest.raises(ValueError):
            factor_device(torch.from_numpy(A).cuda(), 2)
    finally:
        _lib.reset_tuning()


def test_fused_leaves_match_unfused_tree():
    """CAQR_TUNE_FUSE (default 148): R-only TSQR with more than 148 leaves deals the rows
    to at most 148 CTAs in runs of whole 64-row tiles (flat tree inside a CTA, binary tree
    above: the hybrid tree of PAPER.md Fig. 3).  R agrees with the one-CTA-per-leaf binary
    tree and with LAPACK within the R bar; ragged last runs, a tail shorter than n that
    rides with the last run, and 148 < P <= 296 are covered."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    try:
        for (m, n, P) in [(600 * 256, 128, 600), (1000 * 130 + 77, 100, 1000), (297 * 128, 128, 297),
                          (200 * 512, 128, 200), (19205, 100, 150)]:
            A = torch.from_numpy(philox(m).standard_normal((m, n))).cuda()
            _lib.tune(_lib.TUNE_FUSE, 148)
            Rf = factor_device(A, P).R.cpu().numpy()
            assert np.array_equal(Rf, factor_device(A, P).R.cpu().numpy())
            _lib.tune(_lib.TUNE_FUSE, 0)
            R0 = factor_device(A, P).R.cpu().numpy()
            nrm = np.linalg.norm(A.cpu().numpy(), 2)
            assert oracle.r_diff(Rf, R0, nrm) <= 50 * EPS
            assert oracle.r_diff(Rf, np.linalg.qr(A.cpu().numpy(), mode="r"), nrm) <= 1000 * EPS
    finally:
        _lib.reset_tuning()


@pytest.mark.parametrize("m,n,P", [(1500 * 2100, 8, 1500), (4000 * 300 + 123, 8, 4000),
                                   (1300 * 2500 + 3, 5, 1300), (2048 * 1183 + 7, 8, 1200)])
def test_narrow_runs_match_one_warp_per_leaf(m, n, P):
    """CAQR_TUNE_FUSE for n <= 8: with more leaves than 148 x 8 the rows are dealt to
    148 x 8 warps in runs of whole 256-row steps (one wave, flat tree inside a warp, ticket
    tree above).  R agrees with the one-warp-per-leaf tree and with LAPACK; a tail shorter
    than n rides with the last run (last case: 1183 runs of 2048 rows + 7 rows)."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    A = philox(m % 1000 + n).uniform(-1, 1, (m, n))
    At = torch.from_numpy(A).cuda()
    nrm = np.linalg.norm(A, 2)
    try:
        _lib.tune(_lib.TUNE_FUSE, 148)
        Rf = factor_device(At, P).R.cpu().numpy()
        assert np.array_equal(Rf, factor_device(At, P).R.cpu().numpy())
        _lib.tune(_lib.TUNE_FUSE, 0)
        R0 = factor_device(At, P).R.cpu().numpy()
        assert oracle.r_diff(Rf, R0, nrm) <= 50 * EPS
        assert oracle.r_diff(Rf, np.linalg.qr(A, mode="r"), nrm) <= 1000 * EPS
    finally:
        _lib.reset_tuning()


@pytest.mark.parametrize("m,P", [(16384 * 5, 5), (16384 * 3 + 333, 3), (300, 1), (256 * 7 + 1, 2)])
def test_narrow8_parity_and_variants(m, P):
    """CAQR_TUNE_NARROW = 3 (default for contiguous aligned n = 8): 8 rows per
    reflector chain.  R against LAPACK and against the K = 4 kernels (2 / 1),
    ragged last step and short leaves included; misaligned views fall back."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    A = philox(m).uniform(-1, 1, (m, 8))
    At = torch.from_numpy(A).cuda()
    Rl = np.linalg.qr(A, mode="r")
    nrm = np.linalg.norm(A, 2)
    try:
        Rs = {}
        for v in (3, 2, 1):
            _lib.tune(_lib.TUNE_NARROW, v)
            Rs[v] = factor_device(At, P).R.cpu().numpy()
            assert oracle.r_diff(Rs[v], Rl, nrm) <= 1000 * EPS
        _lib.tune(_lib.TUNE_NARROW, 3)
        big = torch.zeros(m * 8 + 1, dtype=torch.float64, device="cuda")
        view = big[1:].view(m, 8)  # 8-byte aligned only: the 8-byte path
        view.copy_(At)
        assert oracle.r_diff(factor_device(view, P).R.cpu().numpy(), Rl, nrm) <= 1000 * EPS
    finally:
        _lib.reset_tuning()


def _dealing_cases():
    rng = np.random.default_rng(20240809)
    cases = []
    for i in range(36):
        wide = i % 2 == 0
        n = int(rng.integers(65, 129)) if wide else int(rng.integers(1, 9))
        P = int(rng.integers(149, 700)) if wide else int(rng.integers(1185, 5000))
        leaf = int(rng.integers(n, 4 * n + 40)) if wide else int(rng.integers(max(n, 16), 700))
        tail = int(rng.integers(0, leaf))
        pad = int(rng.integers(0, 3)) * (1 if i % 3 else 0)  # lda > n for two cases in three
        cases.append((P * leaf + tail, n, P, pad))
    return cases


@pytest.mark.parametrize("m,n,P,pad", _dealing_cases())
def test_row_dealing_random_shapes(m, n, P, pad):
    """R-only TSQR with more leaves than CTA (64 < n <= 128) or warp (n <= 8) slots, seeded
    random shapes: ragged last leaves, leaves barely taller than n, strided views (lda > n).
    The dealt runs give LAPACK's R within the R bar and the one-slot-per-leaf tree's R to a
    few eps, and the same bits on a second call."""
    from paper_0809_2407_b200 import _lib
    from paper_0809_2407_b200.tsqr import factor_device

    A = philox(m + 31 * n + P).standard_normal((m, n + pad))
    At = torch.from_numpy(A).cuda()[:, :n]
    A = A[:, :n]
    nrm = np.linalg.norm(A, 2)
    try:
        Rf = factor_device(At, P).R.cpu().numpy()
        assert np.array_equal(Rf, factor_device(At, P).R.cpu().numpy())
        _lib.tune(_lib.TUNE_FUSE, 0)
        R0 = factor_device(At, P).R.cpu().numpy()
    finally:
        _lib.reset_tuning()
    assert np.array_equal(np.tril(Rf, -1), np.zeros_like(Rf))
    assert oracle.r_diff(Rf, R0, nrm) <= 50 * EPS
    assert oracle.r_diff(Rf, np.linalg.qr(A, mode="r"), nrm) <= 1000 * EPS
