"""Numpy restatement of the TSQR / CAQR compositions (test oracle only).

The reference ships the kernels but not the drivers (tsqr and caqr are
SPEC-only).  The compositions below follow the paper and
the SPEC exactly as SURVEY.md section 8(c) prescribes:

* ``tsqr_reference``: Algorithm 1, reduce variant.  Leaf =
  ``geqr2`` (householder.py:128), combine = ``stacked_qr`` (householder.py:263)
  in ``binary_events`` order (trees.py:52-66,146-152), receiver stacked on top
  (PAPER.md:777-780).
* ``tsqr_reference_q``: the broadcast-like reverse walk.
* ``chain_leaf``: the hybrid leaf the GPU runs:
  a dense first tile (``geqr2``) followed by a flat chain of
  ``tri_rect_qr`` steps (Algorithm 2).
* ``caqr_tsqr``: Algorithm 3 on one process column with
  TSQR panels; its R oracle is ``blocked_qr`` (householder.py:189).
"""

from __future__ import annotations

import numpy as np

from .householder import (
    DimensionError,
    _f64_2d,
    apply_dense,
    apply_stacked,
    apply_tri_rect,
    geqr2,
    stacked_qr,
    tri_rect_qr,
)


def binary_events(P):
    """Combine events (level, receiver, partner) of the binary reduce tree.

    trees.py:52-66 (_binary_levels): at level k pair (f, f + 2^(k-1)) for
    f = 0, 2^k, ... when the partner exists; trees.py:146-152 (schedule):
    level by level, receiver = min of the group.
    """
    if P < 1:
        raise ValueError("P must be >= 1")
    out = []
    k = 1
    while (1 << (k - 1)) < P:
        half = 1 << (k - 1)
        for f in range(0, P, 1 << k):
            if f + half < P:
                out.append((k, f, f + half))
        k += 1
    return out


def block_rows(m, n, P):
    """Row offsets of the 1-D block-row layout (core.py:36-61).

    P blocks of m // P rows, the last one absorbing the remainder; every
    block must have at least n rows (core.py:48-52).
    """
    if P < 1:
        raise DimensionError("P must be >= 1")
    base = m // P
    if base < n:
        raise DimensionError(f"block too short: floor({m}/{P}) = {base} < n = {n}")
    offs = [i * base for i in range(P)] + [m]
    return offs


# --------------------------------------------------------------------------
# reference-semantics TSQR (leaf = dense geqr2)
# --------------------------------------------------------------------------

def tsqr_reference(A, P):
    A = _f64_2d(A)
    m, n = A.shape
    offs = block_rows(m, n, P)
    leaves, Rs = [], []
    for i in range(P):
        Y, tau, R = geqr2(A[offs[i]:offs[i + 1]])
        leaves.append((Y, tau))
        Rs.append(R)
    nodes = []
    for (lvl, a, b) in binary_events(P):
        Yb, tau, R = stacked_qr(Rs[a], Rs[b])
        nodes.append((lvl, a, b, Yb, tau))
        Rs[a] = R
    return {"offs": offs, "leaves": leaves, "nodes": nodes, "R": Rs[0], "n": n}


def _tree_down(nodes, P, n, k):
    S = [None] * P
    S[0] = np.eye(n, k)
    for (lvl, a, b, Yb, tau) in reversed(nodes):
        S[a], S[b] = apply_stacked(Yb, tau, S[a], np.zeros((n, k)))
    return S


def tsqr_reference_q(f):
    offs, n = f["offs"], f["n"]
    P = len(f["leaves"])
    S = _tree_down(f["nodes"], P, n, n)
    Q = np.zeros((offs[-1], n))
    for i, (Y, tau) in enumerate(f["leaves"]):
        C = np.zeros((offs[i + 1] - offs[i], n))
        C[:n] = S[i]
        Q[offs[i]:offs[i + 1]] = apply_dense(Y, tau, C)
    return Q


# --------------------------------------------------------------------------
# hybrid leaf: dense first tile + flat chain of triangle-on-rectangle steps
# --------------------------------------------------------------------------

def chain_tiles(b, h0, ht):
    """(start, stop) row ranges of the leaf chain: dense tile then ht-row tiles."""
    bounds = [(0, min(b, h0))]
    s = min(b, h0)
    while s < b:
        bounds.append((s, min(b, s + ht)))
        s += ht
    return bounds


def chain_leaf(Aleaf, h0, ht):
    """Factor one leaf as the GPU does; returns (tiles, R).

    tiles[0] = (Y0, tau0) dense factor of the first min(b, h0) rows;
    tiles[k] = (V_k, tau_k) triangle-on-rectangle factors of later tiles.
    """
    Aleaf = _f64_2d(Aleaf)
    b, n = Aleaf.shape
    bnds = chain_tiles(b, h0, ht)
    Y0, t0, R = geqr2(Aleaf[bnds[0][0]:bnds[0][1]])
    tiles = [(Y0, t0)]
    for (s, e) in bnds[1:]:
        V, t, R = tri_rect_qr(R, Aleaf[s:e])
        tiles.append((V, t))
    return tiles, R


def chain_leaf_q(tiles, S, b, h0, ht):
    """Rows of Q_leaf [S; 0] (b x k) for a chain leaf; S is n x k."""
    n = tiles[0][0].shape[1]
    k = S.shape[1]
    bnds = chain_tiles(b, h0, ht)
    out = np.zeros((b, k))
    top = np.array(S, dtype=np.float64)
    for (V, t), (s, e) in zip(reversed(tiles[1:]), reversed(bnds[1:])):
        top, out[s:e] = apply_tri_rect(V, t, top, np.zeros((e - s, k)))
    s0, e0 = bnds[0]
    C = np.zeros((e0 - s0, k))
    C[:n] = top
    out[s0:e0] = apply_dense(tiles[0][0], tiles[0][1], C)
    return out


def chain_apply(tiles, C, b, h0, ht, transpose):
    """Q_leaf C or Q_leaf^T C for a chain leaf (C has b rows)."""
    n = tiles[0][0].shape[1]
    C = _f64_2d(C).copy()
    bnds = chain_tiles(b, h0, ht)
    s0, e0 = bnds[0]
    if transpose:
        C[s0:e0] = apply_dense(tiles[0][0], tiles[0][1], C[s0:e0], transpose=True)
        for (V, t), (s, e) in zip(tiles[1:], bnds[1:]):
            C[:n], C[s:e] = apply_tri_rect(V, t, C[:n], C[s:e], transpose=True)
    else:
        for (V, t), (s, e) in zip(reversed(tiles[1:]), reversed(bnds[1:])):
            C[:n], C[s:e] = apply_tri_rect(V, t, C[:n], C[s:e])
        C[s0:e0] = apply_dense(tiles[0][0], tiles[0][1], C[s0:e0])
    return C


def chain_apply_qt(tiles, C, b, h0, ht):
    return chain_apply(tiles, C, b, h0, ht, transpose=True)


def tsqr_hybrid(A, P, h0, ht):
    """TSQR with chain leaves and the binary stacked-triangle tree."""
    A = _f64_2d(A)
    m, n = A.shape
    offs = block_rows(m, n, P)
    leaves, Rs = [], []
    for i in range(P):
        tiles, R = chain_leaf(A[offs[i]:offs[i + 1]], h0, ht)
        leaves.append(tiles)
        Rs.append(R)
    nodes = []
    for (lvl, a, b) in binary_events(P):
        Yb, tau, R = stacked_qr(Rs[a], Rs[b])
        nodes.append((lvl, a, b, Yb, tau))
        Rs[a] = R
    return {"offs": offs, "leaves": leaves, "nodes": nodes, "R": Rs[0], "n": n,
            "h0": h0, "ht": ht, "leaf_R": None}


def tsqr_hybrid_q(f):
    offs, n = f["offs"], f["n"]
    P = len(f["leaves"])
    S = _tree_down(f["nodes"], P, n, n)
    Q = np.zeros((offs[-1], n))
    for i, tiles in enumerate(f["leaves"]):
        b = offs[i + 1] - offs[i]
        Q[offs[i]:offs[i + 1]] = chain_leaf_q(tiles, S[i], b, f["h0"], f["ht"])
    return Q


def tsqr_hybrid_apply(f, C, transpose):
    """Q C (C is n x k thin, or m x k full) or Q^T C (m x k) through the hybrid tree."""
    offs, n = f["offs"], f["n"]
    P = len(f["leaves"])
    if not transpose and np.shape(C)[0] == offs[-1] and offs[-1] != n:
        C = _f64_2d(C).copy()
        for (lvl, a, b, Yb, tau) in reversed(f["nodes"]):
            ra, rb = offs[a], offs[b]
            C[ra:ra + n], C[rb:rb + n] = apply_stacked(Yb, tau, C[ra:ra + n], C[rb:rb + n])
        for i, tiles in enumerate(f["leaves"]):
            b = offs[i + 1] - offs[i]
            C[offs[i]:offs[i + 1]] = chain_apply(tiles, C[offs[i]:offs[i + 1]], b,
                                                 f["h0"], f["ht"], False)
        return C
    if not transpose:
        C = np.asarray(C, dtype=np.float64)
        k = C.shape[1]
        S = [None] * P
        S[0] = C.copy()
        for (lvl, a, b, Yb, tau) in reversed(f["nodes"]):
            S[a], S[b] = apply_stacked(Yb, tau, S[a], np.zeros((n, k)))
        out = np.zeros((offs[-1], k))
        for i, tiles in enumerate(f["leaves"]):
            b = offs[i + 1] - offs[i]
            out[offs[i]:offs[i + 1]] = chain_leaf_q(tiles, S[i], b, f["h0"], f["ht"])
        return out
    C = _f64_2d(C).copy()
    for i, tiles in enumerate(f["leaves"]):
        b = offs[i + 1] - offs[i]
        C[offs[i]:offs[i + 1]] = chain_apply(tiles, C[offs[i]:offs[i + 1]], b,
                                             f["h0"], f["ht"], True)
    for (lvl, a, b, Yb, tau) in f["nodes"]:
        ra, rb = offs[a], offs[b]
        C[ra:ra + n], C[rb:rb + n] = apply_stacked(Yb, tau, C[ra:ra + n], C[rb:rb + n],
                                                   transpose=True)
    return C


# --------------------------------------------------------------------------
# CAQR (Algorithm 3) on one process column, TSQR panels
# --------------------------------------------------------------------------

def caqr_tsqr(A, b, leaf_rows, h0, ht):
    """Right-looking CAQR with hybrid-TSQR panels (Pr = 1).

    Panel j: TSQR of A[jb:, jb:jb+b] over leaves of ``leaf_rows`` rows
    (BlockRowLayout of the active rows), then the leaf-level Q^T update of
    the trailing columns (Alg. 3 line 4) and the tree-level structured
    updates on the leaf top blocks (Alg. 3 lines 5-10, householder.py:335-374).
    Returns (R, panels) with panels[j] the TSQR factor dict of panel j.
    """
    A = _f64_2d(A).copy()
    m, n = A.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    panels = []
    for c0 in range(0, n, b):
        c1 = min(c0 + b, n)
        mj = m - c0
        P = max(1, mj // leaf_rows)
        while P > 1 and mj // P < (c1 - c0):
            P -= 1
        f = tsqr_hybrid(A[c0:, c0:c1], P, h0, ht)
        panels.append(f)
        A[c0:, c0:c1] = 0.0
        A[c0:c0 + (c1 - c0), c0:c1] = f["R"]
        if c1 < n:
            A[c0:, c1:] = tsqr_hybrid_apply(f, A[c0:, c1:], transpose=True)
    return np.triu(A[:n, :n]), panels
