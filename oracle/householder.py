"""Numpy restatement of the reference Householder kernels (test oracle only).

Conventions follow ``pkg/src/caqr/householder.py:9-11``: beta = -sign(x0)*||x||
with sign(0) = +1; a vector already of the form (a, 0, ..., 0) with a >= 0
keeps beta = a and gets tau = 0; (a, 0, ..., 0) with a < 0 gets tau = 2 and
beta = -a.  No overflow scaling (the reference has none).

Matrices are C-ordered float64 (``pkg/src/caqr/core.py:3-5``).
"""

from __future__ import annotations

import numpy as np

EPS = float(np.finfo(np.float64).eps)


class DimensionError(ValueError):
    """Mirror of ``core.DimensionError`` (``pkg/src/caqr/core.py:17-18``)."""


def _f64_2d(a, what="matrix"):
    # pkg/src/caqr/core.py:21-28 (as_matrix): float64, 2-D, finite
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise DimensionError(f"{what} must be 2-D, got ndim={arr.ndim}")
    if arr.size and not np.isfinite(arr).all():
        raise ValueError(f"{what} contains NaN or Inf entries")
    return arr


def reflector(x):
    """(v, tau, beta) with (I - tau v v^T) x = beta e_1, v[0] = 1.

    Follows ``house_gen`` (householder.py:89-114): sigma = ||x[1:]||^2 (:97),
    the three sigma == 0 cases (:101-106), beta = -sign(x0)||x|| (:107-108),
    v[1:] = x[1:] / (x0 - beta) (:110), tau = (beta - x0) / beta (:111).
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size == 0:
        raise DimensionError("reflector needs a nonempty vector")
    v = np.zeros_like(x)
    v[0] = 1.0
    tail = x[1:]
    sig = float(tail @ tail) if x.size > 1 else 0.0
    a = float(x[0])
    if sig == 0.0:
        if a == 0.0:
            return v, 0.0, 0.0
        return (v, 0.0, a) if a >= 0.0 else (v, 2.0, -a)
    nrm = float(np.sqrt(a * a + sig))
    b = nrm if a < 0.0 else -nrm
    v[1:] = tail / (a - b)
    return v, float((b - a) / b), float(b)


def _reflect_cols(block, v, tau):
    # householder.py:117-122 (_update_columns): block := (I - tau v v^T) block
    w = (v @ block) * tau
    block -= np.outer(v, w)


def geqr2(A):
    """Dense Householder QR, column by column -> (Y, tau, R).

    Follows ``qr_unblocked`` (householder.py:128-145): Y is m x n unit lower
    trapezoidal with the unit diagonal stored (:134,138); the update is
    skipped when tau == 0 (:142); R = triu of the top n x n block (:144).
    """
    A = _f64_2d(A).copy()
    m, n = A.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    Y = np.zeros((m, n))
    tau = np.zeros(n)
    for j in range(n):
        v, t, b = reflector(A[j:, j])
        Y[j:, j] = v
        tau[j] = t
        A[j, j] = b
        A[j + 1:, j] = 0.0
        if t != 0.0 and j + 1 < n:
            _reflect_cols(A[j:, j + 1:], v, t)
    return Y, tau, np.triu(A[:n, :n])


def larft(Y, tau):
    """Forward/columnwise T with I - Y T Y^T = H_0 ... H_{n-1}.

    Follows ``form_t`` (householder.py:148-164): T[j,j] = tau_j and
    T[:j,j] = -tau_j T[:j,:j] (Y[j:,:j]^T Y[j:,j]); column skipped if tau_j = 0.
    """
    Y = np.asarray(Y, dtype=np.float64)
    n = Y.shape[1]
    T = np.zeros((n, n))
    for j in range(n):
        T[j, j] = tau[j]
        if j and tau[j] != 0.0:
            z = Y[j:, :j].T @ Y[j:, j]
            T[:j, j] = -tau[j] * (T[:j, :j] @ z)
    return T


def _upper(R, what):
    # householder.py:254-260 (_check_upper_triangular)
    R = _f64_2d(R, what)
    if R.shape[0] != R.shape[1]:
        raise DimensionError(f"{what} must be square, got {R.shape}")
    if np.any(np.tril(R, -1) != 0.0):
        raise DimensionError(f"{what} is not upper triangular")
    return R


def stacked_qr(Ra, Rb):
    """QR of [Ra; Rb] (two n x n upper triangles) on the sparsity profile.

    Follows ``qr_stacked_triangles`` with q = 2 (householder.py:263-294):
    reflector j touches row j of Ra and rows 0..j of Rb (:281-283).
    Returns (Ybot, tau, R): Ybot is the n x n upper-triangular lower block
    of the STACKED factor's Y (the top block is exactly I, test :176-186).
    """
    Ra = _upper(Ra, "triangle 0")
    Rb = _upper(Rb, "triangle 1")
    n = Ra.shape[0]
    if Rb.shape != (n, n):
        raise DimensionError(f"triangle 1 has shape {Rb.shape}, expected {(n, n)}")
    top = Ra.copy()
    bot = Rb.copy()
    Yb = np.zeros((n, n))
    tau = np.zeros(n)
    for j in range(n):
        x = np.concatenate(([top[j, j]], bot[: j + 1, j]))
        v, t, b = reflector(x)
        Yb[: j + 1, j] = v[1:]
        tau[j] = t
        top[j, j] = b
        bot[: j + 1, j] = 0.0
        if t != 0.0 and j + 1 < n:
            blk = np.vstack([top[j:j + 1, j + 1:], bot[: j + 1, j + 1:]])
            _reflect_cols(blk, v, t)
            top[j, j + 1:] = blk[0]
            bot[: j + 1, j + 1:] = blk[1:]
    return Yb, tau, np.triu(top)


def tri_rect_qr(R, B):
    """QR of [R; B] with R upper triangular (n x n) and B rectangular (r x n).

    Follows ``qr_triangle_on_rect`` (householder.py:297-332): reflector j acts
    on row j of R and all rows of B; only the r x n rectangle V is returned
    (implicit identity top).  Returns (V, tau, R_new).
    """
    R = _upper(R, "triangle").copy()
    B = _f64_2d(B, "rectangle").copy()
    n = R.shape[0]
    if B.shape[1] != n:
        raise DimensionError(f"rectangle has {B.shape[1]} columns, triangle has {n}")
    V = np.zeros_like(B)
    tau = np.zeros(n)
    for j in range(n):
        v, t, b = reflector(np.concatenate(([R[j, j]], B[:, j])))
        V[:, j] = v[1:]
        tau[j] = t
        R[j, j] = b
        B[:, j] = 0.0
        if t != 0.0 and j + 1 < n:
            w = (R[j, j + 1:] + v[1:] @ B[:, j + 1:]) * t
            R[j, j + 1:] -= w
            B[:, j + 1:] -= np.outer(v[1:], w)
    return V, tau, R


def apply_dense(Y, tau, C, transpose=False):
    """Q C (or Q^T C) for a DENSE factor, one reflector at a time.

    Follows ``apply_q`` (householder.py:377-391) for the dense row set
    ``reflector(j)`` (:62-64): reverse order for Q, forward for Q^T (:383),
    tau == 0 skipped (:385-386).
    """
    C = _f64_2d(C).copy()
    n = Y.shape[1]
    order = range(n) if transpose else range(n - 1, -1, -1)
    for j in order:
        if tau[j] == 0.0:
            continue
        _reflect_cols(C[j:], Y[j:, j], tau[j])
    return C


def apply_stacked(Yb, tau, Ctop, Cbot, transpose=False):
    """Q [Ctop; Cbot] for a q = 2 STACKED factor (row set householder.py:65-70)."""
    Ct = _f64_2d(Ctop).copy()
    Cb = _f64_2d(Cbot).copy()
    n = Yb.shape[1]
    order = range(n) if transpose else range(n - 1, -1, -1)
    for j in order:
        if tau[j] == 0.0:
            continue
        v = Yb[: j + 1, j]
        w = (Ct[j] + v @ Cb[: j + 1]) * tau[j]
        Ct[j] -= w
        Cb[: j + 1] -= np.outer(v, w)
    return Ct, Cb


def apply_tri_rect(V, tau, Ctop, Cbot, transpose=False):
    """Q [Ctop; Cbot] for a TRI_ON_RECT factor (row set householder.py:71-77)."""
    Ct = _f64_2d(Ctop).copy()
    Cb = _f64_2d(Cbot).copy()
    n = V.shape[1]
    order = range(n) if transpose else range(n - 1, -1, -1)
    for j in order:
        if tau[j] == 0.0:
            continue
        v = V[:, j]
        w = (Ct[j] + v @ Cb) * tau[j]
        Ct[j] -= w
        Cb -= np.outer(v, w)
    return Ct, Cb


def apply_wy(C, Y, T, transpose):
    """C := (I - Y T Y^T)^(T?) C in place (``_apply_yt``, householder.py:175-179)."""
    W = Y.T @ C
    W = (T.T if transpose else T) @ W
    C -= Y @ W


def blocked_qr(A, nb):
    """Right-looking blocked QR (``qr_blocked``, householder.py:189-211).

    Panel ``geqr2`` (:203), ``larft`` (:208), trailing compact-WY Q^T
    update (:209).  The Pr = Pc = 1 degenerate of CAQR.
    Returns (Y, tau, R).
    """
    A = _f64_2d(A).copy()
    m, n = A.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if not 1 <= nb <= n:
        raise DimensionError(f"nb must be in [1, {n}], got {nb}")
    if nb == 1:
        return geqr2(A)
    Y = np.zeros((m, n))
    tau = np.zeros(n)
    for c0 in range(0, n, nb):
        c1 = min(c0 + nb, n)
        Yp, tp, Rp = geqr2(A[c0:, c0:c1])
        Y[c0:, c0:c1] = Yp
        tau[c0:c1] = tp
        A[c0:, c0:c1] = 0.0
        A[c0:c1, c0:c1] = Rp
        if c1 < n:
            apply_wy(A[c0:, c1:], Yp, larft(Yp, tp), transpose=True)
    return Y, tau, np.triu(A[:n, :n])
