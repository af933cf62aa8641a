"""Correction vector v on the device (reference correction.py).

v = sqrt(x s) .* W (ADW)^+ infeas, with (ADW)^+ r = ADW' Q^-1 r applied from
the CholeskyQR2 factor and the hash gather fused with sqrt(x s) (K7).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from .errors import DimensionMismatch, NonpositivePoint, StaleFactor
from .lp_model import reduce_call
from .preconditioning import PreconditionerFactor, apply_pinv_adw, reconstruct
from .runtime import F64, stream_ptr, to_host
from .sketching import SketchOperator


@dataclass
class CorrectionVector:
    """v (device, this rank's entries) and its diagnostics (correction.py:26-38)."""

    v: torch.Tensor
    invariant_residual: float
    norm_bound_slack: float = float("nan")
    _norm: float | None = None

    @property
    def norm(self) -> float:
        return float(self._norm)


def compute_v(f: PreconditionerFactor, W: SketchOperator, x: torch.Tensor, s: torch.Tensor,
              infeas: torch.Tensor, scale: float | None = None, comm=None,
              check_positive: bool = True) -> CorrectionVector:
    """correction.py:41-65. x, s: this rank's entries; infeas: replicated m-vector."""
    if x.shape != s.shape or x.shape[0] != W.n_local:
        raise DimensionMismatch(f"x/s shapes {tuple(x.shape)}/{tuple(s.shape)}, "
                                f"expected ({W.n_local},)")
    if check_positive:
        st = torch.stack([reduce_call("skb_vec_stats", 4, x, None, x.numel())[3],
                          reduce_call("skb_vec_stats", 4, s, None, s.numel())[3]])
        if comm is not None:
            comm.combine_(st, ("min", "min"))
        if not bool((st > 0).all()):
            raise NonpositivePoint("x and s must be strictly positive")
    if f.sketch_tag is not None and f.sketch_tag != W.tag:
        raise StaleFactor(f"factor built from {f.sketch_tag}, got sketch {W.tag}")
    if infeas.shape != (f.m,):
        raise DimensionMismatch(f"infeas has shape {tuple(infeas.shape)}, expected ({f.m},)")
    u = apply_pinv_adw(f, infeas)
    v = torch.empty_like(x)
    if W.kind in ("identity", "gaussian"):
        # v = sqrt(x s) * (W u): W u is u's row slice (identity) or a dense gemv (Gaussian)
        t = W.matvec(u)
        _lib.call("skb_sqrt_xs_scale", t, x, s, v, x.numel(), stream_ptr())
    else:
        _lib.call("skb_sketch_gather", W.cols, W.vals, W.s, x.numel(), u, x, s, v, stream_ptr())
    # ||ADW u - infeas|| / denom   (correction.py:61-64)
    rec = reconstruct(f, u, sub=infeas)
    st = reduce_call("skb_vec_stats", 4, rec, None, f.m)
    vst = reduce_call("skb_vec_stats", 4, v, None, v.numel())
    if comm is not None:
        comm.combine_(vst, ("sum", "sum", "max", "min"))
    inf_norm = None
    if scale is None:
        inf_norm = reduce_call("skb_vec_stats", 4, infeas, None, f.m)
    host = to_host(torch.cat([st, vst] + ([inf_norm] if inf_norm is not None else [])))
    denom = scale if scale is not None else math.sqrt(host[8]) + 1.0
    if denom <= 0.0:
        denom = 1.0
    cv = CorrectionVector(v=v, invariant_residual=math.sqrt(host[0]) / denom)
    cv._norm = math.sqrt(host[4])
    cv.v_sum = float(host[5])
    return cv


def check_v_norm(cv: CorrectionVector, mu: float, f_norm: float, n: int | None = None) -> float:
    """Slack of ||v|| <= sqrt(3 n mu) ||f~|| (correction.py:68-74)."""
    n = cv.v.shape[0] if n is None else n
    slack = float(math.sqrt(3.0 * n * mu) * f_norm - cv.norm)
    cv.norm_bound_slack = slack
    return slack


def check_v_small_enough(cv: CorrectionVector, gamma: float, sigma: float, mu: float) -> bool:
    """||v|| <= gamma sigma mu / 4, inclusive (correction.py:77-80)."""
    return cv.norm <= gamma * sigma * mu / 4.0
