"""Streamed TSQR: the matrix stays in host memory and flows through the GPU in
row chunks (SPEC.md:270-294 ``tsqr_sequential`` / Alg. 2's out-of-core use,
PAPER.md:840-894, 1441).

The leaves are exactly those of the in-HBM path -- ``BlockRowLayout(m, n, P)``
with the same P -- and every chunk holds a power-of-two run of 2^k leaves
starting at a multiple of 2^k, i.e. whole subtrees of the global binary tree.
Each chunk is one ``tsqr_f64_r_binary_rows`` call (leaves + the chunk's
subtree, fused) writing its subtree root into the leaf-indexed R slots; after
the last chunk the remaining binary levels combine the chunk roots
(``tsqr_f64_r_combine_level``: the same combine arithmetic as the fused tree).  The
combine pairs are the same as in ``factor_device`` (trees.py:52-66), so R is
bitwise identical to the device-resident path.

Copy/compute overlap: chunk c+1 is copied host->device on a copy stream into
one of ``buffers`` device buffers while chunk c is factored; a buffer is
reused only after the chunk that last used it is done (events).  Pinned host
tensors are copied directly; other host inputs go through two pinned staging
buffers (a host memcpy per chunk, overlapped with the device work).

Device memory: ``buffers`` chunks + P R slots, independent of m -- matrices
larger than HBM stream through the same kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .core import BlockRowLayout, DimensionError

CHUNK_BYTES = 1 << 30


def plan_chunks(m: int, n: int, P: int, chunk_leaves: int):
    """[(leaf0, leaves, row0, rows)] for chunks of ``chunk_leaves`` (a power of
    two) leaves of BlockRowLayout(m, n, P); the last chunk takes the remainder
    rows with its last leaf."""
    if chunk_leaves < 1 or chunk_leaves & (chunk_leaves - 1):
        raise ValueError("chunk_leaves must be a power of two")
    lay = BlockRowLayout(m, n, P)
    base = lay.base
    out = []
    for l0 in range(0, P, chunk_leaves):
        k = min(chunk_leaves, P - l0)
        r0 = l0 * base
        r1 = m if l0 + k == P else (l0 + k) * base
        out.append((l0, k, r0, r1 - r0))
    return out


def upper_events(P: int, chunk_leaves: int):
    """Binary-tree levels above the chunk subtrees: per level an int32 array of
    (receiver, sender, node id) events (trees.py:52-66 pairs (f, f + 2^(l-1)))."""
    lev = []
    kk = chunk_leaves.bit_length() - 1
    L = max(0, (P - 1).bit_length())
    for l in range(kk + 1, L + 1):
        step = 1 << l
        half = step >> 1
        ev = [(f, f + half, i) for i, f in enumerate(range(0, P, step)) if f + half < P]
        if ev:
            lev.append(np.asarray(ev, dtype=np.int32))
    return lev


def default_chunk_leaves(m: int, n: int, P: int, chunk_bytes: int = CHUNK_BYTES) -> int:
    leaf_bytes = 8 * n * max(1, m // P)
    k = max(1, chunk_bytes // leaf_bytes)
    k = 1 << (int(k).bit_length() - 1)
    return min(k, 1 << max(0, (P - 1).bit_length()))


def tsqr_stream(A, P: int, chunk_leaves: int | None = None, device=None, buffers: int = 3):
    """R (n x n, on the device) of the R-only binary-tree TSQR of the host
    matrix A over P leaves, streamed in chunks (see module doc).

    A: numpy array or CPU torch tensor, row-major (C order) or column-major
    (a Fortran-ordered numpy array, e.g. a memory-mapped MAT1 file --
    ``matio.open_mat1``): column-major chunks are staged as n column
    segments and transposed on the device (``tsqr_f64_colmajor_to_rowmajor``).
    """
    from .tsqr import _check_flag, _ptr

    lib = _lib.load()
    colmajor = False
    if isinstance(A, np.ndarray):
        if A.ndim != 2:
            raise DimensionError("A must be 2-D")
        if A.dtype != np.float64:
            A = A.astype(np.float64)
        if A.flags.f_contiguous and not A.flags.c_contiguous:
            colmajor = True
            An = A
        else:
            At = torch.from_numpy(np.ascontiguousarray(A))
    elif isinstance(A, torch.Tensor):
        if A.is_cuda:
            raise ValueError("tsqr_stream takes a host matrix")
        At = A.to(torch.float64).contiguous()
    else:
        raise TypeError("A must be a numpy array or a CPU torch tensor")
    m, n = A.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    K = chunk_leaves or default_chunk_leaves(m, n, P)
    chunks = plan_chunks(m, n, P, K)
    max_rows = max(c[3] for c in chunks)
    nbuf = max(1, min(buffers, len(chunks)))
    bufs = [torch.empty((max_rows, n), dtype=torch.float64, device=dev) for _ in range(nbuf)]
    pinned = (not colmajor) and At.is_pinned()
    stages = []
    if not pinned:  # host staging (column-major: n column segments per chunk)
        stages = [torch.empty(max_rows * n, dtype=torch.float64, pin_memory=True)
                  for _ in range(min(2, len(chunks)))]
    cm_scratch = torch.empty(max_rows * n, dtype=torch.float64, device=dev) if colmajor else None
    Rs = torch.empty((P, n, n), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    nlev = max(1, (K - 1).bit_length())
    tickets = torch.empty(nlev * K, dtype=torch.int32, device=dev)
    base = m // P
    st = torch.cuda.current_stream(dev)
    cs = torch.cuda.Stream(device=dev)
    done = [None] * nbuf
    staged = [None] * len(stages)
    for c, (l0, k, r0, rows) in enumerate(chunks):
        slot = c % nbuf
        if not pinned:
            si = c % len(stages)
            if staged[si] is not None:
                staged[si].synchronize()  # the H2D that last read this staging buffer is done
            if colmajor:
                # n contiguous column segments (page cache / memmap reads)
                np.copyto(stages[si][:rows * n].numpy().reshape(n, rows), An[r0:r0 + rows].T)
                src = stages[si][:rows * n]
            else:
                stages[si][:rows * n].view(rows, n).copy_(At[r0:r0 + rows])
                src = stages[si][:rows * n].view(rows, n)
        else:
            src = At[r0:r0 + rows]
        if done[slot] is not None:
            cs.wait_event(done[slot])
        with torch.cuda.stream(cs):
            if colmajor:
                cm_scratch[:rows * n].copy_(src, non_blocking=True)
                _lib.check(lib.tsqr_f64_colmajor_to_rowmajor(_ptr(cm_scratch), rows, rows, n,
                                                             _ptr(bufs[slot]), n,
                                                             int(cs.cuda_stream)),
                           "tsqr_f64_colmajor_to_rowmajor")
            else:
                bufs[slot][:rows].copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        if not pinned:
            staged[c % len(stages)] = ev
        st.wait_event(ev)
        _lib.check(lib.tsqr_f64_r_binary_rows(_ptr(bufs[slot]), n, rows, n, k, base,
                                              _ptr(Rs) + 8 * l0 * n * n, _ptr(tickets), _ptr(flag),
                                              int(st.cuda_stream)), "tsqr_f64_r_binary_rows")
        d = torch.cuda.Event()
        d.record(st)
        done[slot] = d
    for e in upper_events(P, K):
        ev_d = torch.from_numpy(e).to(dev)
        _lib.check(lib.tsqr_f64_r_combine_level(_ptr(Rs), n, _ptr(ev_d), len(e),
                                                int(st.cuda_stream)), "tsqr_f64_r_combine_level")
    for b in bufs:
        b.record_stream(cs)
    if cm_scratch is not None:
        cm_scratch.record_stream(cs)
    _check_flag(flag)
    return Rs[0]
