"""Kernel-level Householder API with the reference's names, on the GPU.

Mirrors ``pkg/src/caqr/householder.py``: every
function keeps the reference's signature, return convention ``(factor, R)``,
shape tags and error types, and has no shape limit beyond the reference's own:

* blocks of <= 128 rows and columns -> the single-CTA shared-memory sweep
  ``tsqr_f64_block_factor`` (qr_unblocked, qr_triangle_on_rect,
  qr_stacked_triangles, house_gen);
* anything larger -> ``tsqr_f64_geqr2``, the general in-place geqr2 kernel
  (dense factors; on stacked triangles / [R; B] its exact zeros reproduce the
  structured reflectors);
* qr_blocked -> the reference's algorithm (:189-211): qr_unblocked panels,
  form_t, and the compact-WY trailing update as library GEMMs; nb = 1 is
  qr_unblocked itself, as in the reference (:199-200);
* qr_recursive -> Elmroth-Gustavson recursion (:214-251): the halves
  factored recursively, the left half applied to the right one in compact WY,
  T merged as T12 = -T1 (Y1^T Y2) T2;
* form_t -> Gram by one library GEMM, recurrence ``tsqr_f64_form_t``;
* apply_q / apply_qt / explicit_q / apply_qt_structured -> the block apply
  kernels up to 128 rows, compact WY (I - Y T Y^T) above.

The SPEC drivers (tsqr, caqr) are in ``tsqr`` / ``caqr``.  Inputs may be numpy
(results come back as numpy, like the reference) or CUDA torch tensors.  There
is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import DimensionError
from .counters import FlopCounter, count_geqr2, count_house, count_stacked, count_tri_rect
from .tsqr import _ptr, _stream, _out, to_device

EPS = float(np.finfo(np.float64).eps)
BLOCK_ROWS = 128

DENSE = "dense"
STACKED = "stacked-triangles"
TRI_ON_RECT = "triangle-on-rect"
CHAIN = "chain"
BLOCKED = "blocked"


@dataclass
class HouseholderFactor:
    """Implicit Q = H_0 ... H_{n-1} (householder.py:31-86).

    DENSE: Y m x n unit lower trapezoid; STACKED: Y (q n) x n with the stacked
    profile; TRI_ON_RECT: Y = the r x n rectangle under an implicit identity;
    CHAIN / BLOCKED: multi-tile factors produced by the TSQR / CAQR kernels,
    with Y / tau holding their storage and ``impl`` the device factor.
    """

    Y: np.ndarray
    tau: np.ndarray
    shape_tag: str = DENSE
    q: int = 0
    rows_rect: int = 0
    T: np.ndarray | None = None
    impl: object = field(default=None, repr=False)

    @property
    def n(self) -> int:
        return self.Y.shape[1]

    @property
    def m(self) -> int:
        if self.shape_tag == TRI_ON_RECT:
            return self.n + self.rows_rect
        if self.shape_tag == CHAIN:
            return self.impl.m
        if self.shape_tag == BLOCKED:
            return self.impl.m
        return self.Y.shape[0]

    def reflector(self, j: int):
        """Row indices and values of v_j (householder.py:60-77)."""
        n = self.n
        if self.shape_tag == DENSE:
            return np.arange(j, self.Y.shape[0]), self.Y[j:, j]
        if self.shape_tag == STACKED:
            idx = np.concatenate([[j]] + [np.arange(t * n, t * n + j + 1) for t in range(1, self.q)])
            return idx, self.Y[idx, j]
        if self.shape_tag == TRI_ON_RECT:
            idx = np.concatenate([[j], np.arange(n, n + self.rows_rect)])
            return idx, np.concatenate([[1.0], self.Y[:, j]])
        raise DimensionError(f"{self.shape_tag} factors are not a single reflector set")

    def full_y(self) -> np.ndarray:
        if self.shape_tag == TRI_ON_RECT:
            out = np.zeros((self.m, self.n))
            out[: self.n] = np.eye(self.n)
            out[self.n:] = self.Y
            return out
        if self.shape_tag in (DENSE, STACKED):
            return self.Y
        raise DimensionError(f"{self.shape_tag} factors have no single compact-WY Y")


def _dev(x, like=None):
    dev = like.device if like is not None else torch.device("cuda")
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=dev)


def _flag(dev):
    return torch.zeros(1, dtype=torch.int32, device=dev)


def _check_upper(R, name):
    Rt, host = to_device(R, name=name)
    if Rt.shape[0] != Rt.shape[1]:
        raise DimensionError(f"{name} must be square, got {tuple(Rt.shape)}")
    if bool((torch.tril(Rt, -1) != 0).any()):
        raise DimensionError(f"{name} is not upper triangular")
    if not bool(torch.isfinite(Rt).all()):
        raise ValueError(f"{name} contains NaN or Inf entries")
    return Rt, host


def _block_factor(A: torch.Tensor, n: int, mode: int, R: torch.Tensor):
    lib = _lib.load()
    rows = A.shape[0]
    Y = torch.zeros((rows, n), dtype=torch.float64, device=A.device)
    tau = torch.zeros(n, dtype=torch.float64, device=A.device)
    flag = _flag(A.device)
    _lib.check(lib.tsqr_f64_block_factor(_ptr(A), A.shape[1], rows, n, _ptr(R), _ptr(Y), n,
                                         _ptr(tau), mode, _ptr(flag), _stream(A.device)),
               "tsqr_f64_block_factor")
    if int(flag.item()):
        raise ValueError("matrix contains NaN or Inf entries")
    return Y, tau


# ---------------------------------------------------------------------------
# factorizations
# ---------------------------------------------------------------------------

def house_gen(x, counter: FlopCounter | None = None):
    """(v, tau, beta) with (I - tau v v^T) x = beta e_1 (householder.py:89-114)."""
    xt = torch.as_tensor(np.asarray(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x,
                         dtype=torch.float64)
    if xt.ndim != 1 or xt.numel() == 0:
        raise DimensionError("house_gen expects a nonempty vector")
    L = xt.numel()
    A = xt.to("cuda").reshape(L, 1).contiguous()
    if L <= BLOCK_ROWS:
        R = torch.zeros((1, 1), dtype=torch.float64, device=A.device)
        Y, tau = _block_factor(A, 1, 0, R)
        v = Y[:, 0].clone()
        beta = float(R[0, 0])
    else:
        W, tau = _geqr2(A)
        v = W[:, 0].clone()
        beta = float(W[0, 0])
    v[0] = 1.0
    if counter is not None:
        counter.add(*count_house(L))
    return v.cpu().numpy(), float(tau[0]), beta


def _geqr2(At: torch.Tensor):
    """In-place geqr2 of a copy of At (LAPACK layout) -> (W, tau)."""
    lib = _lib.load()
    W = At.clone().contiguous()
    m, n = W.shape
    tau = torch.zeros(n, dtype=torch.float64, device=W.device)
    flag = _flag(W.device)
    _lib.check(lib.tsqr_f64_geqr2(_ptr(W), n, m, n, _ptr(tau), _ptr(flag), _stream(W.device)),
               "tsqr_f64_geqr2")
    if int(flag.item()):
        raise ValueError("matrix contains NaN or Inf entries")
    return W, tau


def _unit_lower(W: torch.Tensor, n: int) -> torch.Tensor:
    Y = torch.tril(W[:, :n], -1)
    Y[torch.arange(n), torch.arange(n)] = 1.0
    return Y


def _dense_qr(At: torch.Tensor):
    """qr_unblocked on the device: (Y m x n unit lower trapezoid, tau, R)."""
    m, n = At.shape
    if m <= BLOCK_ROWS:
        R = torch.zeros((n, n), dtype=torch.float64, device=At.device)
        Yraw, tau = _block_factor(At.contiguous(), n, 0, R)
        return _unit_lower(Yraw, n), tau, R
    W, tau = _geqr2(At)
    return _unit_lower(W, n), tau, torch.triu(W[:n])


def qr_unblocked(A, counter: FlopCounter | None = None):
    """Householder QR (householder.py:128-145): (DENSE factor, R)."""
    At, host = to_device(A)
    m, n = At.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    Y, tau, R = _dense_qr(At)
    if counter is not None:
        counter.add(*count_geqr2(m, n))
    f = HouseholderFactor(Y.cpu().numpy(), tau.cpu().numpy(), DENSE, impl=(Y, tau))
    return f, _out(R, host)


def _apply_yt(C: torch.Tensor, Y: torch.Tensor, T: torch.Tensor, transpose: bool) -> None:
    """C := (I - Y T Y^T)^(T?) C in place (householder.py:175-186), as GEMMs."""
    W = Y.T @ C
    W = (T.T if transpose else T) @ W
    C -= Y @ W


def _form_t_dev(Y: torch.Tensor, tau: torch.Tensor) -> torch.Tensor:
    lib = _lib.load()
    n = Y.shape[1]
    G = (Y.T @ Y).contiguous()
    T = torch.empty((n, n), dtype=torch.float64, device=Y.device)
    if n <= 512:
        _lib.check(lib.tsqr_f64_form_t(_ptr(G), n, n, _ptr(tau), _ptr(T), n, _stream(Y.device)),
                   "tsqr_f64_form_t")
        return T
    # T = D (I + S D)^-1 with S = striu(G), D = diag(tau): the recurrence in closed form
    D = torch.diag(tau)
    U = torch.eye(n, dtype=torch.float64, device=Y.device) + torch.triu(G, 1) @ D
    return torch.linalg.solve_triangular(U, D, upper=True, left=False, unitriangular=True)


def qr_blocked(A, nb: int, counter: FlopCounter | None = None):
    """Blocked QR (householder.py:189-211): qr_unblocked panels of width nb,
    trailing update through each panel's T; nb = 1 is qr_unblocked itself."""
    At, host = to_device(A)
    m, n = At.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if not 1 <= nb <= n:
        raise DimensionError(f"nb must be in [1, {n}], got {nb}")
    if nb == 1:
        return qr_unblocked(A, counter)
    W = At.clone()
    Y = torch.zeros((m, n), dtype=torch.float64, device=W.device)
    tau = torch.zeros(n, dtype=torch.float64, device=W.device)
    for j0 in range(0, n, nb):
        j1 = min(j0 + nb, n)
        Yp, tp, Rp = _dense_qr(W[j0:, j0:j1])
        Y[j0:, j0:j1] = Yp
        tau[j0:j1] = tp
        W[j0:, j0:j1] = 0.0
        W[j0:j1, j0:j1] = Rp
        if j1 < n:
            _apply_yt(W[j0:, j1:], Yp, _form_t_dev(Yp, tp), transpose=True)
        if counter is not None:
            counter.add(*count_geqr2(m - j0, j1 - j0))
    R = torch.triu(W[:n, :n])
    f = HouseholderFactor(Y.cpu().numpy(), tau.cpu().numpy(), DENSE, impl=(Y, tau))
    return f, _out(R, host)


def qr_recursive(A, min_width: int = 4, counter: FlopCounter | None = None):
    """Recursive QR (householder.py:214-251): halving column splits, T merged
    on the way up (T12 = -T1 (Y1^T Y2) T2); the factor carries T."""
    At, host = to_device(A)
    m, n = At.shape
    if m < n:
        raise DimensionError(f"need m >= n, got {m} x {n}")
    if min_width < 1:
        raise DimensionError("min_width must be >= 1")
    W = At.clone()

    def rec(block: torch.Tensor):
        bm, bn = block.shape
        if bn <= min_width:
            Yb, tb, Rb = _dense_qr(block)
            block.zero_()
            block[:bn] = Rb
            if counter is not None:
                counter.add(*count_geqr2(bm, bn))
            return Yb, tb, _form_t_dev(Yb, tb)
        n1 = bn // 2
        Y1, t1, T1 = rec(block[:, :n1])
        _apply_yt(block[:, n1:], Y1, T1, transpose=True)
        Y2, t2, T2 = rec(block[n1:, n1:])
        Yb = torch.zeros((bm, bn), dtype=torch.float64, device=block.device)
        Yb[:, :n1] = Y1
        Yb[n1:, n1:] = Y2
        Tb = torch.zeros((bn, bn), dtype=torch.float64, device=block.device)
        Tb[:n1, :n1] = T1
        Tb[n1:, n1:] = T2
        Tb[:n1, n1:] = -T1 @ ((Y1[n1:].T @ Y2) @ T2)
        return Yb, torch.cat([t1, t2]), Tb

    Y, tau, T = rec(W)
    R = torch.triu(W[:n, :n])
    f = HouseholderFactor(Y.cpu().numpy(), tau.cpu().numpy(), DENSE, T=T.cpu().numpy(),
                          impl=(Y, tau))
    return f, _out(R, host)


def qr_stacked_triangles(Rs, counter: FlopCounter | None = None):
    """QR of q stacked n x n upper triangles on the sparsity profile (:263-294)."""
    if len(Rs) < 2:
        raise DimensionError("need at least two stacked triangles")
    q = len(Rs)
    tris = []
    host = False
    for t, R in enumerate(Rs):
        Rt, h = _check_upper(R, f"triangle {t}")
        tris.append(Rt)
        host |= h
    n = tris[0].shape[0]
    for t, R in enumerate(tris):
        if tuple(R.shape) != (n, n):
            raise DimensionError(f"triangle {t} has shape {tuple(R.shape)}, expected {(n, n)}")
    if (q - 1) * n <= BLOCK_ROWS:
        Rtop = tris[0].clone()
        low = torch.cat(tris[1:], dim=0).contiguous()
        Yl, tau = _block_factor(low, n, 3, Rtop)
        Y = torch.cat([torch.eye(n, dtype=torch.float64, device=Yl.device), Yl], dim=0)
    else:  # dense geqr2 of the stack: its exact zeros keep the stacked profile
        Wst, tau = _geqr2(torch.cat(tris, dim=0))
        Y = _unit_lower(Wst, n)
        Rtop = torch.triu(Wst[:n])
    if counter is not None:
        f_, d_ = count_stacked(n, q)
        counter.add(f_, d_)
    f = HouseholderFactor(Y.cpu().numpy(), tau.cpu().numpy(), STACKED, q=q, impl=(Y, tau))
    return f, _out(Rtop, host)


def qr_triangle_on_rect(Rtri, B, counter: FlopCounter | None = None):
    """QR of [R; B] with R triangular (householder.py:297-332)."""
    Rt, host = _check_upper(Rtri, "triangle")
    Bt, h2 = to_device(B, name="rectangle")
    n, r = Rt.shape[0], Bt.shape[0]
    if Bt.shape[1] != n:
        raise DimensionError(f"rectangle has {Bt.shape[1]} columns, triangle has {n}")
    if r <= BLOCK_ROWS and n <= BLOCK_ROWS:
        Rw = Rt.clone()
        Y, tau = _block_factor(Bt, n, 2, Rw)
    else:  # dense geqr2 of [R; B]: zeros below R's diagonal keep the identity top
        Wst, tau = _geqr2(torch.cat([Rt, Bt], dim=0))
        Y = Wst[n:].contiguous()
        Rw = torch.triu(Wst[:n])
    if counter is not None:
        counter.add(*count_tri_rect(n, r))
    f = HouseholderFactor(Y.cpu().numpy(), tau.cpu().numpy(), TRI_ON_RECT, rows_rect=r,
                          impl=(Y, tau))
    return f, _out(Rw, host or h2)


def form_t(Y, tau, counter: FlopCounter | None = None):
    """T with I - Y T Y^T = H_0 ... H_{n-1} (householder.py:148-164): the Gram
    Y^T Y as one library GEMM, the recurrence in ``tsqr_f64_form_t``."""
    Yt = torch.as_tensor(np.asarray(Y) if not isinstance(Y, torch.Tensor) else Y,
                         dtype=torch.float64).to("cuda")
    tt = torch.as_tensor(np.asarray(tau) if not isinstance(tau, torch.Tensor) else tau,
                         dtype=torch.float64).to(Yt.device).contiguous()
    T = _form_t_dev(Yt, tt)
    return T.cpu().numpy() if not isinstance(Y, torch.Tensor) else T


def factor_t(factor: HouseholderFactor, counter: FlopCounter | None = None):
    if factor.T is not None:
        return factor.T
    return form_t(factor.full_y(), factor.tau, counter)


# ---------------------------------------------------------------------------
# applications
# ---------------------------------------------------------------------------

def _block_apply(Y, tau, rows, n, C, mode, transpose, Ctop=None):
    lib = _lib.load()
    k = C.shape[1]
    _lib.check(lib.tsqr_f64_block_apply(_ptr(Y), n, rows, n, _ptr(tau), _ptr(Ctop),
                                        0 if Ctop is None else Ctop.shape[1], _ptr(C), k, k, mode,
                                        int(transpose), _stream(C.device)), "tsqr_f64_block_apply")


def apply_q(factor: HouseholderFactor, C, transpose: bool = False,
            counter: FlopCounter | None = None):
    """Q C (or Q^T C); C has factor.m rows (householder.py:377-391)."""
    Ct, host = to_device(C, name="C")
    if Ct.shape[0] != factor.m:
        raise DimensionError(f"C has {Ct.shape[0]} rows, factor acts on {factor.m}")
    if not bool(torch.isfinite(Ct).all()):
        raise ValueError("C contains NaN or Inf entries")
    tag = factor.shape_tag
    out = Ct.clone()
    n = factor.n
    big = factor.m > BLOCK_ROWS or n > BLOCK_ROWS or (tag == STACKED and factor.q != 2)
    if tag in (DENSE, STACKED, TRI_ON_RECT) and big:
        # compact WY: Q = I - Y T Y^T (T cached on the factor)
        if factor.T is None:
            factor.T = form_t(factor.full_y(), factor.tau)
        Yf = _dev(factor.full_y(), out)
        _apply_yt(out, Yf, _dev(factor.T, out), transpose)
    elif tag == DENSE:
        Y, tau = factor.impl if factor.impl is not None else (_dev(factor.Y), _dev(factor.tau))
        _block_apply(Y.contiguous(), tau, factor.m, n, out, 0, transpose)
    elif tag == TRI_ON_RECT:
        Y, tau = factor.impl if factor.impl is not None else (_dev(factor.Y), _dev(factor.tau))
        top = out[:n].contiguous()
        bot = out[n:].contiguous()
        _block_apply(Y.contiguous(), tau, factor.rows_rect, n, bot, 2, transpose, Ctop=top)
        out = torch.cat([top, bot], dim=0)
    elif tag == STACKED:
        Y, tau = factor.impl if factor.impl is not None else (_dev(factor.Y), _dev(factor.tau))
        lib = _lib.load()
        ev = torch.tensor([[0, 1, 0]], dtype=torch.int32, device=out.device)
        Yb = Y[n:].contiguous()
        _lib.check(lib.tsqr_f64_tree_apply_level(_ptr(Yb), _ptr(tau), n, _ptr(ev), 1, _ptr(out),
                                                 out.shape[1], n, out.shape[1], int(transpose), 0,
                                                 _stream(out.device)), "tsqr_f64_tree_apply_level")
    elif tag == CHAIN:
        from .tsqr import apply_q_device

        out = apply_q_device(factor.impl, Ct, transpose)
    elif tag == BLOCKED:
        from .caqr import caqr_apply_q

        return caqr_apply_q(factor.impl, C, transpose)
    else:
        raise DimensionError(f"unknown factor shape {tag!r}")
    if counter is not None:
        counter.add(4 * factor.m * n * Ct.shape[1])
    return _out(out, host)


def apply_qt(factor: HouseholderFactor, C, counter: FlopCounter | None = None):
    return apply_q(factor, C, transpose=True, counter=counter)


def explicit_q(factor: HouseholderFactor, thin: bool = True):
    m = factor.m
    k = factor.n if thin else m
    E = torch.zeros((m, k), dtype=torch.float64, device="cuda")
    E[:k, :k] = torch.eye(k, dtype=torch.float64, device="cuda")
    return apply_q(factor, E.cpu().numpy())


def apply_qt_structured(factor: HouseholderFactor, T, C0, C1, counter: FlopCounter | None = None):
    """Q^T [C0; C1] for identity-top factors (householder.py:335-374)."""
    if factor.shape_tag == STACKED:
        if factor.q != 2:
            raise DimensionError("inner-product update needs exactly two stacked blocks")
        rows1 = factor.n
    elif factor.shape_tag == TRI_ON_RECT:
        rows1 = factor.rows_rect
    else:
        raise DimensionError("factor has no identity-top structure")
    C0t, h0 = to_device(C0, name="C0")
    C1t, h1 = to_device(C1, name="C1")
    n = factor.n
    if C0t.shape[0] != n:
        raise DimensionError(f"C0 must have {n} rows, got {C0t.shape[0]}")
    if C1t.shape[0] != rows1:
        raise DimensionError(f"C1 must have {rows1} rows, got {C1t.shape[0]}")
    if C0t.shape[1] != C1t.shape[1]:
        raise DimensionError("C0 and C1 must have the same column count")
    both = torch.cat([C0t, C1t], dim=0)
    out = apply_q(factor, both, transpose=True, counter=counter)
    return _out(out[:n], h0 or h1), _out(out[n:], h0 or h1)
