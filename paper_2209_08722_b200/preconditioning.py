"""Sketched preconditioner factor on the device (reference preconditioning.py).

The reference takes a thin SVD of ADW (LAPACK gesdd, preconditioning.py:46)
and applies Q^-1 = U diag(sigma^-2) U' and (ADW)^+ = V diag(sigma^-1) U'.
Here Q = ADW ADW' = L L' comes from CholeskyQR2 on X = ADW' (FP64 DMMA
GEMMs, csrc/skb_dense.cu), so

    apply_inv(f, r)      = Linv' (Linv r)          two triangular gemvs
    apply_pinv_adw(f, r) = X (Linv' (Linv r))      = ADW' Q^-1 r = (ADW)^+ r

which equal the reference's operators whenever ADW has full row rank (the
only case the reference lets through).

Rank test (rank_check): the reference raises RankDeficient when
sigma_min/sigma_max of ADW is below 1e-12 (preconditioning.py:47-50). ADW
and L share their singular values (Q = ADW ADW' = L L'), so the same ratio
is decided from the factor, two-sided:
  * upper bounds of the ratio (below the tolerance => deficient): the
    diagonal ratio min|L_ii| / max|L_ii|, and, when needed, the converged
    power-iteration estimates of lambda_max(Q) and lambda_max(Q^-1)
    (Rayleigh quotients approach the extremes from below);
  * a lower bound (at or above the tolerance => full rank):
    1 / (||L||_F ||L^-1||_F), with ||L||_F = ||ADW||_F. It is within a factor
    m of the true ratio, so the power iterations run only in that gray band.
A Cholesky breakdown that survives the shifted CholeskyQR3 retry is reported
the same way.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import RankDeficient
from .kernels import DeviceMatrix
from .runtime import F64, stream_ptr, to_host, workspace

RANK_TOL = 1e-12


@dataclass
class PreconditionerFactor:
    """Device factor of Q = ADW ADW' (replaces the U/sigma/V_hat triple)."""

    Linv: torch.Tensor    # (Mp, Mp) lower, L^-1
    LinvT: torch.Tensor   # (Mp, Mp) upper, L^-T
    Lfac: torch.Tensor | None  # (Mp, Mp) lower L, only when requested
    X: DeviceMatrix       # ADW' (w x m, bucket-major)
    m: int
    diag_min: float
    diag_max: float
    shifted: bool
    sketch_tag: tuple | None = None
    dist: tuple | None = None   # (w_total, r0, comm): X holds bucket rows [r0, r0 + X.n)

    @property
    def ld(self) -> int:
        return int(self.Linv.shape[1])

    @property
    def w(self) -> int:
        return self.dist[0] if self.dist is not None else self.X.n


def build_preconditioner(X: DeviceMatrix, rank_tol: float = RANK_TOL,
                         sketch_tag: tuple | None = None) -> PreconditionerFactor:
    """Factor ADW (given as X = ADW'); raises RankDeficient like the reference."""
    if getattr(X, "dist", None) is not None:
        return _build_distributed(X, rank_tol, sketch_tag)
    m, w = X.m, X.n
    if w < m:
        raise RankDeficient(f"sketch width {w} below row count {m}")
    Mp = int(_lib.lib().skb_factor_padded_dim(m))
    dev = X.cols.device
    Linv = torch.empty((Mp, Mp), dtype=F64, device=dev)
    LinvT = torch.empty((Mp, Mp), dtype=F64, device=dev)
    Lfac = None  # L itself is not needed by the solver (diag(L) comes from the factor stats)
    need = int(_lib.lib().skb_factor_workspace_bytes(m, w))
    ws, cap = workspace(need)
    stats = np.zeros(4, dtype=np.float64)
    _lib.call("skb_factor_cholqr2", X.cols, X.lda, w, m, Linv, LinvT, Lfac, stats.ctypes.data, ws,
              cap, stream_ptr())
    dmin, dmax, shifted, status = stats
    if int(status) & 4 or not (dmax > 0.0) or not np.isfinite(dmin) or dmin / dmax < rank_tol:
        raise RankDeficient(
            f"ADW numerically rank deficient: diagonal ratio {dmin / max(dmax, 1e-300):.3e}")
    f = PreconditionerFactor(Linv, LinvT, Lfac, X, m, float(dmin), float(dmax), bool(shifted),
                             sketch_tag)
    rank_check(f, rank_tol)
    return f


def _adwt(f: PreconditionerFactor, z: torch.Tensor) -> torch.Tensor:
    """ADW' z for this rank's buckets (w_local-vector)."""
    u = torch.empty(f.X.n, dtype=F64, device=z.device)
    if f.X.n > 0:
        _lib.call("skb_rowdot_gemv", f.X.cols, f.X.lda, f.X.n, f.m, 0, z, u, None, stream_ptr())
    return u


def _q_apply(f: PreconditionerFactor, z: torch.Tensor) -> torch.Tensor:
    """Q z = ADW (ADW' z), ranks' bucket blocks summed."""
    u = _adwt(f, z)
    if f.dist is None:
        from . import kernels as K
        out = torch.empty(f.m, dtype=F64, device=z.device)
        K.gemv(f.X, u, out)
        return out
    w_total, r0, comm = f.dist
    full = torch.zeros(w_total, dtype=F64, device=z.device)
    full[r0:r0 + f.X.n] = u
    return reconstruct(f, full)


def _lambda_max(apply, m: int, dev, max_iter: int = 300, rtol: float = 1e-9) -> float:
    """Largest eigenvalue of an SPD operator by power iteration from a fixed
    start (deterministic); the Rayleigh quotients increase toward it."""
    g = torch.Generator(device=dev)
    g.manual_seed(20220918)
    v = torch.randn(m, dtype=F64, device=dev, generator=g)
    v /= torch.linalg.vector_norm(v)
    lam = 0.0
    for _ in range(max_iter):
        w = apply(v)
        new = float(torch.dot(v, w).item())
        nrm = torch.linalg.vector_norm(w)
        if not (new > 0.0) or not np.isfinite(new):
            return new
        v = w / nrm
        if abs(new - lam) <= rtol * new:
            return new
        lam = new
    return lam


def sigma_ratio_bounds(f: PreconditionerFactor, exact: bool = False):
    """(lower, upper) bounds of sigma_min/sigma_max of ADW from the factor;
    exact=True tightens the upper bound with converged power iterations."""
    m = f.m
    dev = f.Linv.device
    x_fro = (torch.linalg.vector_norm(f.X.cols[:, :m]) ** 2).reshape(1) if f.X.n > 0 else \
        torch.zeros(1, dtype=F64, device=dev)
    if f.dist is not None:
        f.dist[2].allreduce_(x_fro)
    l_fro = torch.linalg.vector_norm(f.Linv[:m, :m]) ** 2
    fx, fl = (float(v) for v in to_host(torch.cat([x_fro.reshape(1), l_fro.reshape(1)])))
    lower = 1.0 / np.sqrt(fx * fl) if fx > 0 and fl > 0 else 0.0
    upper = f.diag_min / f.diag_max if f.diag_max > 0 else 0.0
    if exact:
        lq = _lambda_max(lambda v: _q_apply(f, v), m, dev)
        lqi = _lambda_max(lambda v: apply_inv(f, v), m, dev)
        if lq > 0 and lqi > 0:
            upper = min(upper, 1.0 / np.sqrt(lq * lqi))
    return lower, upper


def rank_check(f: PreconditionerFactor, rank_tol: float = RANK_TOL) -> None:
    """RankDeficient iff sigma_min/sigma_max(ADW) < rank_tol (preconditioning.py:47-50)."""
    lower, upper = sigma_ratio_bounds(f)
    if upper < rank_tol:
        raise RankDeficient(f"ADW numerically rank deficient: sigma ratio <= {upper:.3e}")
    if lower >= rank_tol:
        return
    lower, upper = sigma_ratio_bounds(f, exact=True)
    if upper < rank_tol:
        raise RankDeficient(f"ADW numerically rank deficient: sigma ratio ~ {upper:.3e}")


def _gemm(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower, ws, cap):
    _lib.call("skb_gemm", ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower, 1, 0, 0,
              0, ws, cap, stream_ptr())


def _build_distributed(X: DeviceMatrix, rank_tol: float, sketch_tag) -> PreconditionerFactor:
    """CholeskyQR2 of a bucket-row-distributed X = ADW': every
    rank forms its block's Gram X_g'X_g, the m x m Grams are allreduced, the
    Cholesky / triangular inverse run redundantly on the (identical) sum, and
    Y_g = X_g L1^-T stays local — the O(w m^2) GEMM work is split across ranks,
    only m x m matrices move. Same algorithm and fallback (shifted CholeskyQR3)
    as skb_factor_cholqr2."""
    w_total, r0, comm = X.dist
    m, wb = X.m, X.n
    if w_total < m:
        raise RankDeficient(f"sketch width {w_total} below row count {m}")
    Mp = int(_lib.lib().skb_factor_padded_dim(m))
    dev = X.cols.device
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(m, max(wb, 1))))
    status = torch.zeros(1, dtype=torch.int32, device=dev)

    def gram(Z):
        G = torch.zeros((Mp, Mp), dtype=F64, device=dev)
        if wb > 0:
            _gemm(1, 0, m, m, wb, 1.0, Z.cols, Z.lda, Z.cols, Z.lda, 0.0, G, Mp, 1, ws, cap)
        comm.allreduce_(G)
        _lib.call("skb_set_identity_pad", G, Mp, m, Mp, stream_ptr())
        return G

    def chol(G):
        status.zero_()
        _lib.call("skb_potrf", G, Mp, Mp, status, ws, cap, stream_ptr())
        return int(to_host(status.reshape(-1)[:1])[0])

    G = gram(X)
    shifted = False
    if chol(G) & 4:  # shifted CholeskyQR: s = 11 (m w + m (m + 1)) u ||X||_F^2
        shifted = True
        fro = (X.cols[:, :m] * X.cols[:, :m]).sum().reshape(1)
        comm.allreduce_(fro)
        shift = 11.0 * (m * w_total + m * (m + 1)) * 1.1102230246251565e-16 * float(to_host(fro.reshape(-1)[:1])[0])
        G = gram(X)
        G.diagonal()[:m] += shift
        if chol(G) & 4:
            raise RankDeficient("Cholesky failed after the shifted CholeskyQR retry")
    dprod = G.diagonal()[:m].abs().clone()
    L1i = torch.empty((Mp, Mp), dtype=F64, device=dev)
    _lib.call("skb_trtri", G, L1i, Mp, Mp, ws, cap, stream_ptr())
    Linv = torch.zeros((Mp, Mp), dtype=F64, device=dev)
    Y = DeviceMatrix(torch.zeros_like(X.cols), m)
    for p in range(2 if shifted else 1):
        if wb > 0:  # Y = X L1i' (local rows)
            _gemm(0, 1, wb, m, m, 1.0, X.cols, X.lda, L1i, Mp, 0.0, Y.cols, Y.lda, 0, ws, cap)
        G2 = gram(Y)
        if chol(G2) & 4:
            raise RankDeficient("second CholeskyQR pass lost positive definiteness")
        dprod = dprod * G2.diagonal()[:m].abs()
        L2i = torch.empty((Mp, Mp), dtype=F64, device=dev)
        _lib.call("skb_trtri", G2, L2i, Mp, Mp, ws, cap, stream_ptr())
        Linv.zero_()
        _gemm(0, 0, Mp, Mp, Mp, 1.0, L2i, Mp, L1i, Mp, 0.0, Linv, Mp, 1, ws, cap)
        if p == 0 and shifted:
            L1i = Linv.clone()
    LinvT = torch.empty_like(Linv)
    _lib.call("skb_transpose", Linv, LinvT, Mp, Mp, stream_ptr())
    dstat = to_host(torch.stack([dprod.min(), dprod.max()]))
    dmin, dmax = float(dstat[0]), float(dstat[1])
    if not (dmax > 0.0) or not np.isfinite(dmin) or dmin / dmax < rank_tol:
        raise RankDeficient(
            f"ADW numerically rank deficient: diagonal ratio {dmin / max(dmax, 1e-300):.3e}")
    f = PreconditionerFactor(Linv, LinvT, None, X, m, dmin, dmax, shifted, sketch_tag,
                             dist=X.dist)
    rank_check(f, rank_tol)
    return f


def _tri_gemv(M: torch.Tensor, m: int, tri: int, x: torch.Tensor, y: torch.Tensor, gate=None):
    _lib.call("skb_rowdot_gemv", M, M.shape[1], m, m, tri, x, y, gate, stream_ptr())


def apply_inv(f: PreconditionerFactor, r: torch.Tensor, out: torch.Tensor | None = None,
              tmp: torch.Tensor | None = None) -> torch.Tensor:
    """Q^-1 r = Linv' (Linv r)  (preconditioning.py:59-61)."""
    tmp = torch.empty(f.m, dtype=F64, device=r.device) if tmp is None else tmp
    out = torch.empty(f.m, dtype=F64, device=r.device) if out is None else out
    _tri_gemv(f.Linv, f.m, 1, r, tmp)
    _tri_gemv(f.LinvT, f.m, 2, tmp, out)
    return out


def apply_pinv_adw(f: PreconditionerFactor, r: torch.Tensor) -> torch.Tensor:
    """(ADW)^+ r = ADW' Q^-1 r, a length-w vector (preconditioning.py:64-66)."""
    z = apply_inv(f, r)
    nb = f.X.n
    u = torch.empty(nb, dtype=F64, device=r.device)
    if nb > 0:
        _lib.call("skb_rowdot_gemv", f.X.cols, f.X.lda, nb, f.m, 0, z, u, None, stream_ptr())
    if f.dist is not None:  # bucket blocks -> the whole u on every rank
        u = f.dist[2].allgather_rows(u, f.dist[0])
    return u


def reconstruct(f: PreconditionerFactor, u: torch.Tensor, sub=None) -> torch.Tensor:
    """ADW u [- sub] (= U diag(sigma) V_hat' u, correction.py:61), one pass over X."""
    from . import kernels as K
    out = torch.empty(f.m, dtype=F64, device=u.device)
    if f.dist is None:
        K.gemv(f.X, u, out, sub=sub)
        return out
    w_total, r0, comm = f.dist
    if f.X.n > 0:
        K.gemv(f.X, u[r0:r0 + f.X.n].contiguous(), out)
    else:
        out.zero_()
    comm.allreduce_(out)
    if sub is not None:
        out -= sub
    return out
