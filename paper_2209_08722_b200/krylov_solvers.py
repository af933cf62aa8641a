"""Normal operator and preconditioned CG on the device (reference krylov_solvers.py).

NormalOperator.apply is the fused single-pass A (d^2 .* (A' v)) (K4). pcg
enqueues the whole t_max-step recurrence with no host round trip: on one GPU
as a single libskb call (skb_pcg_solve), under column sharding as a gated
launch sequence with an NCCL allreduce of the matvec between kernels. The
host reads the trace once.
"""

from __future__ import annotations

import threading

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import Breakdown, NonpositiveScaling
from .lp_model import DeviceLP, reduce_call
from .preconditioning import PreconditionerFactor, apply_inv
from .runtime import F64, stream_ptr, to_host, workspace


class NormalOperator:
    """Matrix-free A D^2 A' with D = diag(d) (krylov_solvers.py:28-50).

    lp: DeviceLP (this rank's columns); d: device vector of the local
    columns. d2 may be supplied precomputed (skb_step_prep makes both)."""

    def __init__(self, lp: DeviceLP, d: torch.Tensor, d2: torch.Tensor | None = None,
                 check: bool = True):
        if tuple(d.shape) != (lp.n_local,):
            raise ValueError(f"d has shape {tuple(d.shape)}, expected ({lp.n_local},)")
        if check and lp.vec_stats(d)[3] <= 0.0:
            raise NonpositiveScaling("d must be strictly positive")
        self.lp = lp
        self.d = d
        self._d2 = d * d if d2 is None else d2

    @property
    def m(self) -> int:
        return self.lp.m

    def apply(self, v, out=None, sub=None, gate=None):
        """A (d^2 .* (A' v)) [- sub]; numpy in -> numpy out (host round trip)."""
        host = not isinstance(v, torch.Tensor)
        if host:
            v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(self.lp.device)
        r = self.lp.normal(self._d2, v, out=out, sub=sub, gate=gate)
        return r.cpu().numpy() if host else r


@dataclass
class SolverTrace:
    """Residual history of one inner solve (krylov_solvers.py:53-62)."""

    residual_norms: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    zeta: float | None = None
    t_max: int = 0


class _PcgBuffers:
    """Per-m scratch reused across PCG calls (vectors, state, trace)."""

    def __init__(self, m: int, t_cap: int, device):
        self.m, self.t_cap = m, t_cap
        self.ldv = ((m + 31) // 32) * 32
        self.vec = torch.empty(5 * self.ldv, dtype=F64, device=device)
        nb = int(_lib.lib().skb_pcg_state_bytes())
        self.state = torch.zeros((nb + 7) // 8, dtype=F64, device=device)
        self.trace = torch.zeros(t_cap + 1, dtype=F64, device=device)
        self.trace_host = np.zeros(t_cap + 1, dtype=np.float64)
        self.out_host = np.zeros(3, dtype=np.int32)

    def v(self, k):
        return self.vec[k * self.ldv:k * self.ldv + self.m]


# Per-thread (run_comparison runs solves from a thread pool, oracle_bench.py:236):
# PCG state, trace and host readback buffers are never shared between solves.
_BUF = threading.local()


def _buffers(m: int, t_max: int, device) -> _PcgBuffers:
    cache = getattr(_BUF, "d", None)
    if cache is None:
        cache = _BUF.d = {}
    key = (device.index, m)
    b = cache.get(key)
    if b is None or b.t_cap < t_max:
        b = cache[key] = _PcgBuffers(m, max(t_max, 64), device)
    return b


def _raise_status(status: int, where: str):
    if status & 1:
        raise Breakdown(f"nonpositive curvature in {where}")
    if status & 2:
        raise Breakdown("preconditioner produced a negative inner product")


def pcg(op, f: PreconditionerFactor, p: torch.Tensor, t_max: int, tol: float):
    """Preconditioned CG on A D^2 A' dy = p with M^-1 = Q^-1 (krylov_solvers.py:65-105).

    Returns (dy device tensor, SolverTrace). Raises Breakdown on nonpositive
    curvature or a negative r'Q^-1 r, like the reference."""
    m = op.m
    dev = p.device
    t_max = int(t_max)
    B = _buffers(m, t_max, dev)
    dy = torch.empty(m, dtype=F64, device=dev)
    lp = getattr(op, "lp", None)
    if isinstance(op, NormalOperator) and not lp.comm.active and not lp.sparse:
        ws, cap = workspace(int(_lib.lib().skb_stream_workspace_bytes(m)))
        _lib.call("skb_pcg_solve", lp.A.cols, m, lp.A.n, lp.A.lda, op._d2, f.Linv, f.LinvT, f.ld,
                  p, dy, B.vec, B.ldv, t_max, float(tol), B.state, B.trace,
                  B.trace_host.ctypes.data, B.out_host.ctypes.data, ws, cap, stream_ptr())
        iters, conv, status = (int(v) for v in B.out_host)
    else:
        iters, conv, status = _pcg_generic(op, f, p, dy, t_max, tol, B)
    _raise_status(status, "pcg")
    norms = [float(v) for v in B.trace_host[:iters + 1]]
    return dy, SolverTrace(residual_norms=norms, iterations=iters, converged=bool(conv),
                           t_max=t_max)


def _pcg_generic(op, f, p, dy, t_max, tol, B):
    """Launch-sequence PCG for sharded or duck-typed operators. Sharded
    NormalOperators run gated (no host sync per iteration); other operators
    are checked on the host after every step, like the reference loop."""
    m = op.m
    sp_ = stream_ptr()
    r, z, q, Aq, t = (B.v(k) for k in range(5))
    gate = B.state  # PcgState.stop is the first int after four doubles
    stop_ptr = B.state.data_ptr() + 32
    _lib.call("skb_pcg_init", p, r, dy, m, B.state, sp_)
    apply_inv(f, r, out=z, tmp=t)
    _lib.call("skb_pcg_init2", r, z, q, m, float(tol), B.state, B.trace, sp_)
    gated = isinstance(op, NormalOperator)
    state_view = B.state.view(torch.int32)
    for _ in range(t_max):
        if not gated:
            if int(to_host(state_view[8:9])[0]):  # stop flag (host check per step)
                break
            Aq.copy_(op.apply(q))
        else:
            op.apply(q, out=Aq, gate=_Ptr(stop_ptr))
        _lib.call("skb_pcg_step_a", q, Aq, dy, r, m, B.state, sp_)
        _lib.call("skb_rowdot_gemv", f.Linv, f.ld, m, m, 1, r, t, _Ptr(stop_ptr), sp_)
        _lib.call("skb_rowdot_gemv", f.LinvT, f.ld, m, m, 2, t, z, _Ptr(stop_ptr), sp_)
        _lib.call("skb_pcg_step_b", r, z, q, m, t_max, B.state, B.trace, sp_)
    st = to_host(state_view[8:12])
    iters, conv, status = int(st[2]), int(st[3]), int(st[1])
    n = iters + 1
    B.trace_host[:n] = to_host(B.trace[:n])
    return iters, conv, status


def _state_result(B):
    st = to_host(B.state.view(torch.int32)[8:12])
    iters, conv, status = int(st[2]), int(st[3]), int(st[1])
    B.trace_host[:iters + 1] = to_host(B.trace[:iters + 1])
    return iters, conv, status


def _apply_step(op, q, Aq, stop_ptr, state_view):
    """Aq = op(q): gated device launch for NormalOperator, host-checked otherwise.
    Returns False when a foreign operator's loop should end (state stopped)."""
    if isinstance(op, NormalOperator):
        op.apply(q, out=Aq, gate=_Ptr(stop_ptr))
        return True
    if int(to_host(state_view[8:9])[0]):
        return False
    Aq.copy_(op.apply(q))
    return True


def chebyshev(op, f: PreconditionerFactor, p: torch.Tensor, zeta: float, t_max: int,
              tol: float | None = None):
    """Chebyshev iteration on the fixed band [2/(2+zeta), 2/(2-zeta)]
    (krylov_solvers.py:108-153). Returns (dy, SolverTrace)."""
    from .errors import InvalidZeta
    if not 0.0 < zeta <= 1.0:
        raise InvalidZeta(f"zeta must lie in (0, 1], got {zeta}")
    lam_min = 2.0 / (2.0 + zeta)
    lam_max = 2.0 / (2.0 - zeta)
    d0 = 0.5 * (lam_max + lam_min)
    c = 0.5 * (lam_max - lam_min)
    m = op.m
    t_max = int(t_max)
    B = _buffers(m, t_max, p.device)
    dy = torch.empty(m, dtype=F64, device=p.device)
    r, z, q, Aq, t = (B.v(k) for k in range(5))
    sp_ = stream_ptr()
    stop_ptr = B.state.data_ptr() + 32
    state_view = B.state.view(torch.int32)
    _lib.call("skb_pcg_init", p, r, dy, m, B.state, sp_)
    apply_inv(f, r, out=z, tmp=t)
    _lib.call("skb_cheb_init", r, z, m, float(tol) if tol is not None else -1.0, B.state,
              B.trace, sp_)
    alpha = 0.0
    for k in range(t_max):
        if k == 0:
            alpha, beta = 1.0 / d0, 0.0
        else:
            beta = (0.5 if k == 1 else 0.25) * (c * alpha) ** 2
            alpha = 1.0 / (d0 - beta / alpha)
        _lib.call("skb_cheb_step_q", z, q, dy, m, alpha, beta, 1 if k == 0 else 0, B.state, sp_)
        if not _apply_step(op, q, Aq, stop_ptr, state_view):
            break
        _lib.call("skb_cheb_step_r", r, Aq, m, alpha, B.state, sp_)
        _lib.call("skb_rowdot_gemv", f.Linv, f.ld, m, m, 1, r, t, _Ptr(stop_ptr), sp_)
        _lib.call("skb_rowdot_gemv", f.LinvT, f.ld, m, m, 2, t, z, _Ptr(stop_ptr), sp_)
        _lib.call("skb_cheb_trace", r, z, m, t_max, B.state, B.trace, sp_)
    iters, conv, _ = _state_result(B)
    if tol is None:
        conv = 1
    norms = [float(v) for v in B.trace_host[:iters + 1]]
    return dy, SolverTrace(residual_norms=norms, iterations=iters, converged=bool(conv),
                           zeta=zeta, t_max=t_max)


def unpreconditioned_cg(op, p: torch.Tensor, t_max: int, tol: float):
    """Plain CG baseline; the trace holds ||r|| (krylov_solvers.py:174-204).
    The PCG kernels run with z aliased to r (M = I)."""
    m = op.m
    t_max = int(t_max)
    B = _buffers(m, t_max, p.device)
    dy = torch.empty(m, dtype=F64, device=p.device)
    r, _, q, Aq, _ = (B.v(k) for k in range(5))
    sp_ = stream_ptr()
    stop_ptr = B.state.data_ptr() + 32
    state_view = B.state.view(torch.int32)
    _lib.call("skb_pcg_init", p, r, dy, m, B.state, sp_)
    _lib.call("skb_pcg_init2", r, r, q, m, float(tol), B.state, B.trace, sp_)
    for _ in range(t_max):
        if not _apply_step(op, q, Aq, stop_ptr, state_view):
            break
        _lib.call("skb_pcg_step_a", q, Aq, dy, r, m, B.state, sp_)
        _lib.call("skb_pcg_step_b", r, r, q, m, t_max, B.state, B.trace, sp_)
    iters, conv, status = _state_result(B)
    _raise_status(status, "unpreconditioned_cg")
    norms = [float(v) for v in B.trace_host[:iters + 1]]
    return dy, SolverTrace(residual_norms=norms, iterations=iters, converged=bool(conv),
                           t_max=t_max)


DIRECT_CAP = 2000


def direct_solve(op: "NormalOperator", p: torch.Tensor, cap: int = DIRECT_CAP) -> torch.Tensor:
    """Dense Cholesky of A D^2 A' with one refinement pass (krylov_solvers.py:156-171):
    DMMA weighted Gram, blocked device Cholesky, triangular inverse."""
    from .errors import NotPositiveDefinite, TooLarge
    m = op.m
    if m > cap:
        raise TooLarge(f"m={m} exceeds direct-solve cap {cap}")
    lp = op.lp
    Mp = int(_lib.lib().skb_factor_padded_dim(m))
    dev = p.device
    G = torch.zeros((Mp, Mp), dtype=F64, device=dev)
    ws, cap_b = workspace(int(_lib.lib().skb_factor_workspace_bytes(m, m)))
    Ad = lp.dense_A()
    _lib.call("skb_weighted_gram", Ad.cols, m, Ad.n, Ad.lda, op._d2, G, Mp, ws, cap_b, stream_ptr())
    if lp.comm.active:
        lp.comm.allreduce_(G)
    _lib.call("skb_set_identity_pad", G, Mp, m, Mp, stream_ptr())
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("skb_potrf", G, Mp, Mp, status, ws, cap_b, stream_ptr())
    if int(to_host(status.reshape(-1)[:1])[0]) & 4:
        raise NotPositiveDefinite("Cholesky of the normal matrix failed")
    Linv = torch.empty_like(G)
    _lib.call("skb_trtri", G, Linv, Mp, Mp, ws, cap_b, stream_ptr())
    LinvT = torch.empty_like(G)
    _lib.call("skb_transpose", Linv, LinvT, Mp, Mp, stream_ptr())

    class _F:  # the two-gemv Q^-1 application on the exact normal matrix
        pass
    fac = _F()
    fac.Linv, fac.LinvT, fac.m = Linv, LinvT, m
    dy = apply_inv(fac, p)
    resid = op.apply(dy)
    _lib.call("skb_sub", p, resid, resid, m, stream_ptr())   # resid = p - A D^2 A' dy
    corr = apply_inv(fac, resid)
    _lib.call("skb_axpy", dy, 1.0, corr, dy, m, stream_ptr())
    return dy


class _Ptr:
    """A raw device address passed through _lib.call as a pointer."""

    def __init__(self, addr: int):
        self.addr = addr

    def data_ptr(self):
        return self.addr
