"""Strictly feasible start construction on the device (reference ipm_core.py:806-969,
lp_model.py:206-239): phase 1, shifted-objective dual point, centering prelude.

Every stage reuses the hot path: the auxiliary LPs are solved by the device
`solve`, the centering step is a sketched PCG + correction + fused direction
pass, and the step-length grid / ratio tests are reductions over n-vectors.
Only scalars (step lengths, thresholds) are decided on the host.
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .distributed import MIN, SUM  # noqa: F401
from .errors import DegenerateRow, Infeasible, InvariantViolated, MaxIterations
from .errors import NeighborhoodViolated, NotPositiveDefinite, Unbounded
from .lp_model import DeviceLP, LinearProgram, reduce_call
from .runtime import F64, stream_ptr, workspace

V_INVARIANT_TOL = 1e-10
FEAS_TOL = 1e-9


def _sub_params(params, **overrides):
    """Auxiliary solves: infeasible mode, auto sketch sizes, diagnostics off (:806-811)."""
    base = replace(params, mode="infeasible", w=None, s=None, t_max=None, diag_cond=False,
                   max_outer=max(params.max_outer, 400))
    return replace(base, **overrides)


def phase1_lp(lp: DeviceLP):
    """min 1'z s.t. A_f x + z = b_f, (x, z) >= 0 with rows sign-flipped so b_f > 0
    (lp_model.py:206-239). Returns (aux DeviceLP, start iterate).

    The auxiliary matrix [A_f, I] keeps A's storage: a CSC A gets a CSC
    auxiliary (A's entries, sign-flipped, then one entry per identity column --
    never densified), a dense A a column-major copy. Under column sharding each
    rank keeps its block of A_f and the m identity columns go to the last rank,
    so rank blocks stay contiguous and in order."""
    from .ipm_core import make_iterate
    from .kernels import DeviceMatrix, SparseDeviceMatrix
    b = lp.b
    sign = torch.where(b < 0, -1.0, 1.0).to(F64)
    bf = sign * b
    zero = torch.nonzero(bf == 0.0)
    if zero.numel():
        raise DegenerateRow(int(zero[0, 0].item()))
    m, n = lp.m, lp.n
    dev = lp.device
    comm = lp.comm
    last = comm.rank == comm.world - 1
    nl = lp.n_local
    nid = m if last else 0                      # identity columns held here
    if lp.sparse:
        A = lp.A
        base = A.colptr[0]
        cp = A.colptr - base
        nnz = int(cp[-1].item())
        rows = A.rowidx[int(base.item()):int(base.item()) + nnz]
        vals = A.vals[int(base.item()):int(base.item()) + nnz] * sign[rows.long()]
        if nid:
            cp = torch.cat([cp, nnz + torch.arange(1, m + 1, dtype=torch.int64, device=dev)])
            rows = torch.cat([rows, torch.arange(m, dtype=torch.int32, device=dev)])
            vals = torch.cat([vals, torch.ones(m, dtype=F64, device=dev)])
        Aaux = SparseDeviceMatrix(cp.contiguous(), rows.contiguous(), vals.contiguous(), m)
        Af = A  # A_f 1 = sign .* (A 1): the row sign is applied to the sums below
    else:
        lda = lp.A.lda
        cols = torch.zeros((nl + nid, lda), dtype=F64, device=dev)
        cols[:nl, :m].copy_(lp.A.cols[:, :m] * sign[None, :])  # A_f = diag(sign) A
        if nid:
            cols[nl + torch.arange(m, device=dev), torch.arange(m, device=dev)] = 1.0
        Aaux = DeviceMatrix(cols, m)
        Af = DeviceMatrix(cols[:nl], m)
    c_aux = torch.cat([torch.zeros(nl, dtype=F64, device=dev),
                       torch.ones(nid, dtype=F64, device=dev)])
    aux = DeviceLP.from_device(Aaux, bf.contiguous(), c_aux, n + m, j0=lp.j0, comm=comm,
                               name=lp.name + "_phase1")
    from . import kernels as K
    ones = torch.ones(nl, dtype=F64, device=dev)
    row_sums = torch.empty(m, dtype=F64, device=dev)
    if nl > 0:
        K.gemv(Af, ones, row_sums)                                   # A_f 1 (local block)
    else:
        row_sums.zero_()
    if lp.sparse:
        row_sums = row_sums * sign
    comm.allreduce_(row_sums)
    top = float(row_sums.max().item())
    eps = float(bf.min().item() / (2.0 * top)) if top > 0 else 1.0
    bh, rh = bf.cpu().numpy(), row_sums.cpu().numpy()
    z = bh - eps * rh
    while not np.all(z > 0):
        eps *= 0.5
        z = bh - eps * rh
    x = np.concatenate([np.full(n, eps), z])
    y = np.zeros(m)
    s = np.maximum(np.concatenate([np.zeros(n), np.ones(m)]) + 1.0, 1.0)
    return aux, make_iterate(aux, x, y, s)


def _pcg_solve_aat(lp: DeviceLP, rhs: torch.Tensor, params) -> torch.Tensor:
    """(A A')^-1 rhs without forming A A' (sparse or sharded A): PCG on the
    normal operator with D = I, preconditioned by the sketched factor of A
    itself -- the hot path with d = 1 -- to 1e-14 relative."""
    from .ipm_core import _build_factor
    from .krylov_solvers import NormalOperator, pcg
    from .sketching import auto_sketch_dims
    ones = torch.ones(lp.n_local, dtype=F64, device=lp.device)
    op = NormalOperator(lp, ones, check=False)
    w, s_nnz = auto_sketch_dims(lp.m, lp.n, params.delta)
    w = min(lp.n, max(4 * lp.m, min(w, 8 * lp.m)))
    rng = np.random.Generator(np.random.Philox(int(params.seed) + 0x5EED))
    W, factor, _ = _build_factor(lp, ones, params, rng, w, max(4, min(s_nnz, 8)))
    y, trace = pcg(op, factor, rhs, max(200, 4 * lp.m), 1e-14)
    return y


def _chol_solve_aat(lp: DeviceLP, rhs: torch.Tensor) -> torch.Tensor:
    """(A A')^-1 rhs on the device (dense Cholesky of A A', ipm_core.py:836-839)."""
    m = lp.m
    Mp = int(_lib.lib().skb_factor_padded_dim(m))
    G = torch.zeros((Mp, Mp), dtype=F64, device=lp.device)
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(m, m)))
    ones = torch.ones(lp.n_local, dtype=F64, device=lp.device)
    Ad = lp.dense_A()
    _lib.call("skb_weighted_gram", Ad.cols, m, Ad.n, Ad.lda, ones, G, Mp, ws, cap, stream_ptr())
    lp.comm.allreduce_(G)
    _lib.call("skb_set_identity_pad", G, Mp, m, Mp, stream_ptr())
    status = torch.zeros(1, dtype=torch.int32, device=lp.device)
    _lib.call("skb_potrf", G, Mp, Mp, status, ws, cap, stream_ptr())
    if int(status.item()) & 4:
        raise NotPositiveDefinite("A A' not positive definite")
    Li = torch.empty_like(G)
    _lib.call("skb_trtri", G, Li, Mp, Mp, ws, cap, stream_ptr())
    LiT = torch.empty_like(G)
    _lib.call("skb_transpose", Li, LiT, Mp, Mp, stream_ptr())
    t = torch.empty(m, dtype=F64, device=lp.device)
    out = torch.empty(m, dtype=F64, device=lp.device)
    _lib.call("skb_rowdot_gemv", Li, Mp, m, m, 1, rhs, t, None, stream_ptr())
    _lib.call("skb_rowdot_gemv", LiT, Mp, m, m, 2, t, out, None, stream_ptr())
    return out


def phase1_point(lp: DeviceLP, params):
    """Strictly positive x0 with A x0 = b (ipm_core.py:814-846) -> (x0, aux report)."""
    from .ipm_core import solve
    params.validate()
    aux, aux_start = phase1_lp(lp)
    rep = solve(aux, start=aux_start, params=_sub_params(params, tol_outer=1e-10))
    z_sum = float(np.sum(rep.x[lp.n:]))
    if z_sum > 1e-7 * (1.0 + lp.b_norm):
        raise Infeasible(f"phase-1 optimum 1'z = {z_sum:.3e} is bounded away from zero")
    x0 = lp.local(torch.from_numpy(np.ascontiguousarray(rep.x[:lp.n])).to(lp.device))
    if lp.sparse:  # all-zero columns: x = 1 (ipm_core.py:831-832)
        x0[(lp.A.colptr[1:] - lp.A.colptr[:-1]) == 0] = 1.0
    elif lp.n_local > 0:
        _lib.call("skb_zero_col_fill", lp.A.cols, lp.m, lp.A.n, lp.A.lda, x0, stream_ptr())
    from .errors import Breakdown, RankDeficient
    try:
        resid = lp.gemv(x0, sub=lp.b)                 # A x0 - b
        resid.neg_()                                  # b - A x0
        if lp.sparse or lp.comm.active:               # never densify A (c4) or gather it
            y = _pcg_solve_aat(lp, resid, params)
        else:
            y = _chol_solve_aat(lp, resid)
        corr = lp.gemv_t(y)                           # A' (A A')^-1 (b - A x0)
        cand = x0 + corr
        cmin = torch.tensor([float(cand.min().item()) if cand.numel() else float("inf")],
                            dtype=F64, device=lp.device)
        lp.comm.allreduce_(cmin, MIN)
        if float(cmin.item()) > 0:
            x0 = cand
    except (NotPositiveDefinite, Breakdown, RankDeficient):
        pass
    xmin = torch.tensor([float(x0.min().item()) if x0.numel() else float("inf")],
                        dtype=F64, device=lp.device)
    lp.comm.allreduce_(xmin, MIN)
    if not float(xmin.item()) > 0:
        raise NeighborhoodViolated("phase-1 produced a boundary primal point")
    return x0, rep


def _centering_step(lp: DeviceLP, it, params, rng):
    """One sigma = 1 Newton step with the centrality-maximising length (:914-969)."""
    from .correction import compute_v
    from .ipm_core import _build_factor, _candidate, assemble_directions, build_rhs, \
        default_t_max
    from .krylov_solvers import NormalOperator, pcg
    from .sketching import auto_sketch_dims
    d, d2 = lp.new_n(), lp.new_n()
    reduce_call("skb_step_prep", 3, it.x, it.s, it.x.numel(), d, d2)
    op = NormalOperator(lp, d, d2=d2, check=False)
    p = build_rhs(lp, it, 1.0, "feasible")
    p_norm = lp.norm_m(p)
    w, s_nnz = auto_sketch_dims(lp.m, lp.n, params.delta)
    if params.w is not None:
        w = params.w
    if params.s is not None:
        s_nnz = params.s
    t_budget = max(40, 4 * default_t_max(lp.n, params))
    last = float("inf")
    for _ in range(3):
        W, factor, _r = _build_factor(lp, d, params, rng, w, s_nnz)
        dy, _t = pcg(op, factor, p, t_budget, 1e-13)
        infeas = op.apply(dy, sub=p)
        scale = lp.norm_m(infeas) + p_norm
        cv = compute_v(factor, W, it.x, it.s, infeas, scale=scale if scale > 0 else 1.0,
                       comm=lp.comm, check_positive=False)
        last = lp.norm_m(lp.gemv_ratio(cv.v, it.s, sub=infeas)) / max(scale, 1e-300)
        if last <= V_INVARIANT_TOL:
            break
    else:
        raise InvariantViolated(f"centering correction off by {last:.3e}")
    dirn = assemble_directions(lp, it, dy, cv.v, 1.0, "feasible")
    rm = reduce_call("skb_ratio_min", 2, it.x, dirn.dx, it.s, dirn.ds, it.x.numel())
    lp.comm.combine_(rm, (MIN, MIN))
    a_hi = 1.0
    for v in rm.cpu().numpy():
        if np.isfinite(v):
            a_hi = min(a_hi, 0.9999 * float(v))
    if a_hi <= 0.0:
        raise NeighborhoodViolated("centering step blocked at the boundary")
    grid = np.linspace(0.0, a_hi, 65)[1:]
    best_alpha, best_theta = 0.0, it.min_xs / it.mu
    stats = []
    for k0 in range(0, 64, 8):
        al = torch.from_numpy(np.ascontiguousarray(grid[k0:k0 + 8])).to(lp.device)
        st = reduce_call("skb_centering_grid", 24, it.x, it.s, dirn.dx, dirn.ds, al,
                         it.x.numel())
        lp.comm.combine_(st, tuple([MIN, SUM, SUM] * 8))
        stats.append(st)
    h = torch.cat(stats).cpu().numpy().reshape(64, 3)
    for a, (mn, sm, nonpos) in zip(grid, h):
        if nonpos > 0:
            continue
        theta = float(mn / (sm / lp.n))
        if theta > best_theta:
            best_alpha, best_theta = float(a), theta
    if best_alpha == 0.0:
        raise NeighborhoodViolated("centering step made no centrality progress")
    new = _candidate(lp, it, dirn, best_alpha)
    new.k = it.k + 1
    if (new.rp_norm > FEAS_TOL * (1.0 + lp.b_norm) or new.rd_norm > FEAS_TOL * (1.0 + lp.c_norm)):
        raise InvariantViolated("centering step drifted off the feasible set")
    return new


def feasible_start(lp: DeviceLP, params):
    """Phase 1 -> shifted dual -> centering prelude -> mu to O(1) (ipm_core.py:849-911)."""
    from .ipm_core import IpmIterate, default_start, ipm_step, make_iterate, solve
    from .kernels import DeviceMatrix
    params.validate()
    rng = np.random.Generator(np.random.Philox(int(params.seed) + 0x9E3779B9))
    x0, _ = phase1_point(lp, params)
    y0 = s0 = None
    c_scale = 1.0 + float(lp.vec_stats(lp.c)[2])
    for delta in (1e-2 * c_scale, 1e-4 * c_scale, 1e-6 * c_scale):
        shifted = DeviceLP.from_device(lp.A, lp.b, lp.c - delta, lp.n, lp.j0, lp.comm,
                                       name=lp.name + "_shifted")
        try:
            rep = solve(shifted, start=default_start(shifted),
                        params=_sub_params(params, tol_outer=1e-10, max_outer=200))
        except (MaxIterations, Unbounded):
            continue
        y_cand = torch.from_numpy(np.ascontiguousarray(rep.y)).to(lp.device)
        s_cand = lp.gemv_t(y_cand)                          # A' y
        s_cand = lp.c - s_cand                              # c - A' y
        smin = torch.tensor([float(s_cand.min().item()) if s_cand.numel() else float("inf")],
                            dtype=F64, device=lp.device)
        lp.comm.allreduce_(smin, MIN)
        if float(smin.item()) >= 0.25 * delta:
            y0, s0 = y_cand, s_cand
            break
    if y0 is None:
        raise Unbounded("no interior dual point found: dual feasible region appears to have "
                        "empty interior")
    it = make_iterate(lp, x0, y0, s0)
    target = min(0.99, 1.05 * (1.0 - params.gamma))
    for _ in range(50):
        if it.min_xs / it.mu >= target:
            break
        it = _centering_step(lp, it, params, rng)
    else:
        raise NeighborhoodViolated("centering prelude failed to reach N(gamma)")
    shrink = replace(params, mode="feasible", w=None, s=None, t_max=None, diag_cond=False)
    for _ in range(300):
        if it.mu <= 1.0:
            break
        it, _ = ipm_step(lp, it, shrink, rng)
    it.k = 0
    return it
