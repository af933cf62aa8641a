"""Sketched preconditioner factor on the device (reference preconditioning.py).

The reference takes a thin SVD of ADW (LAPACK gesdd, preconditioning.py:46)
and applies Q^-1 = U diag(sigma^-2) U' and (ADW)^+ = V diag(sigma^-1) U'.
Here Q = ADW ADW' = L L' comes from CholeskyQR2 on X = ADW' (FP64 DMMA
GEMMs, csrc/skb_dense.cu), so

    apply_inv(f, r)      = Linv' (Linv r)          two triangular gemvs
    apply_pinv_adw(f, r) = X (Linv' (Linv r))      = ADW' Q^-1 r = (ADW)^+ r

which equal the reference's operators whenever ADW has full row rank (the
only case the reference lets through). Rank test: the reference raises
RankDeficient when sigma_min/sigma_max < 1e-12; since sigma_min(L) <=
min|L_ii| and sigma_max(L) >= max|L_ii|, a diagonal ratio below the
tolerance proves deficiency, and a Cholesky breakdown that survives the
shifted CholeskyQR3 retry is reported the same way.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import RankDeficient
from .kernels import DeviceMatrix
from .runtime import F64, stream_ptr, workspace

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

    @property
    def ld(self) -> int:
        return int(self.Linv.shape[1])

    @property
    def w(self) -> int:
        return self.X.n


def build_preconditioner(X: DeviceMatrix, rank_tol: float = RANK_TOL,
                         sketch_tag: tuple | None = None) -> PreconditionerFactor:
    """Factor ADW (given as X = ADW'); raises RankDeficient like the reference."""
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
    return PreconditionerFactor(Linv, LinvT, Lfac, X, m, float(dmin), float(dmax), bool(shifted),
                                sketch_tag)


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
    u = torch.empty(f.w, dtype=F64, device=r.device)
    _lib.call("skb_rowdot_gemv", f.X.cols, f.X.lda, f.w, f.m, 0, z, u, None, stream_ptr())
    return u


def reconstruct(f: PreconditionerFactor, u: torch.Tensor, sub=None) -> torch.Tensor:
    """ADW u [- sub] (= U diag(sigma) V_hat' u, correction.py:61), one pass over X."""
    from . import kernels as K
    out = torch.empty(f.m, dtype=F64, device=u.device)
    K.gemv(f.X, u, out, sub=sub)
    return out
