"""ORACLE — test infrastructure only (see oracle/__init__.py).

numpy/scipy restatement of the reference's sketch -> factor -> PCG ->
correction -> step path. Every routine names the reference lines it restates
(paths relative to /root/reference/pkg/src/skipm). The restatement keeps the
reference's floating-point operation order so that, on the same inputs, it
reproduces the reference bit for bit; tests/test_oracle_golden.py checks this
against fixtures produced by the live reference (tests/golden/make_golden.py).

Scope: solver="pcg" with sparse-sign, identity or Gaussian sketches, both
modes, correction on. Start construction (feasible_start / phase1_point) and
zero-cost circulation rebalancing (ipm_core.py:737-803) are not restated: the
benchmark configurations supply their own start and have no zero-cost columns.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

# ipm_core.py:61-67
FEAS_TOL = 1e-9
PROXIMITY_SLACK = 1e-12
RATIO_FLOOR = 1e-32
RATIO_CAP = 1e32
V_INVARIANT_TOL = 1e-10
MU_IDENTITY_TOL = 1e-10
DIRECTION_TOL = 1e-8
RANK_TOL = 1e-12  # preconditioning.py:19


class OracleError(Exception):
    """Raised where the reference raises; .kind names the reference class."""

    def __init__(self, kind: str, msg: str = ""):
        self.kind = kind
        super().__init__(f"{kind}: {msg}")


# --------------------------------------------------------------- sketching


def philox(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(int(seed)))


def auto_sketch_dims(m: int, n: int, delta: float):
    """sketching.py:83-90."""
    lg = max(1, math.ceil(math.log2(m / delta)))
    w = min(n, 8 * m * lg)
    return w, min(max(2, lg), w)


def sparse_embedding(n: int, w: int, s: int, seed: int):
    """sketching.py:93-119 -> (cols int64 (n,s), vals f64 (n,s))."""
    if not (1 <= s <= w) or w > n * s:
        raise OracleError("InvalidDims", f"n={n} w={w} s={s}")
    g = philox(seed)
    if 2 * s >= w:
        cols = np.argsort(g.random((n, w)), axis=1)[:, :s].copy()
    else:
        cols = g.integers(0, w, size=(n, s))
        while True:
            srt = np.sort(cols, axis=1)
            bad = (np.diff(srt, axis=1) == 0).any(axis=1)
            if not bad.any():
                break
            cols[bad] = g.integers(0, w, size=(int(bad.sum()), s))
    vals = (g.integers(0, 2, size=(n, s)) * 2.0 - 1.0) / math.sqrt(s)
    return cols, vals


def gaussian_sketch(n: int, w: int, seed: int) -> np.ndarray:
    """sketching.py:131-139."""
    return philox(seed).standard_normal((n, w)) / math.sqrt(w)


class Sketch:
    """Minimal stand-in for SketchOperator (sketching.py:31-80)."""

    def __init__(self, kind, n, w, s, seed, cols=None, vals=None, dense=None):
        self.kind, self.n, self.w, self.s, self.seed = kind, n, w, s, seed
        self.cols, self.vals, self.dense = cols, vals, dense

    def as_csr(self):
        if self.kind == "identity":
            return sp.identity(self.n, format="csr")
        ptr = np.arange(0, self.n * self.s + 1, self.s)
        csr = sp.csr_matrix((self.vals.ravel().copy(), self.cols.ravel().copy(), ptr),
                            shape=(self.n, self.w))
        csr.sort_indices()
        return csr

    def matvec(self, u):
        if self.kind == "identity":
            return u.copy()
        if self.kind == "gaussian":
            return self.dense @ u
        return np.sum(self.vals * u[self.cols], axis=1)


def apply_sketch(A: sp.csr_matrix, d: np.ndarray, W: Sketch) -> np.ndarray:
    """sketching.py:142-161 (ADW, dense m x w)."""
    if not np.all(d > 0):
        raise OracleError("NonpositiveScaling")
    AD = A.multiply(d[None, :]).tocsr()
    if W.kind == "identity":
        return np.asarray(AD.toarray())
    if W.kind == "gaussian":
        return np.asarray(AD @ W.dense)
    return np.asarray((AD @ W.as_csr()).toarray())


# --------------------------------------------------------- preconditioner


class Factor:
    """preconditioning.py:22-35 (thin SVD of ADW)."""

    def __init__(self, ADW, tag=None):
        ADW = np.asarray(ADW, dtype=np.float64)
        m, w = ADW.shape
        if w < m:
            raise OracleError("RankDeficient", "w < m")
        U, sig, Vt = np.linalg.svd(ADW, full_matrices=False)   # preconditioning.py:46
        if sig[0] <= 0.0 or sig[-1] / sig[0] < RANK_TOL:       # preconditioning.py:47
            raise OracleError("RankDeficient", f"{sig[-1] / max(sig[0], 1e-300):.3e}")
        self.U, self.sig, self.Vh, self.tag = U, sig, Vt.T, tag

    @property
    def m(self):
        return self.U.shape[0]

    def inv(self, r):          # preconditioning.py:59-61
        return self.U @ ((self.U.T @ r) / self.sig**2)

    def pinv(self, r):         # preconditioning.py:64-66
        return self.Vh @ ((self.U.T @ r) / self.sig)


# ------------------------------------------------------ normal op and PCG


class NormalOp:
    """krylov_solvers.py:28-50: v -> A (d^2 * (A' v))."""

    def __init__(self, A, d):
        if not np.all(d > 0):
            raise OracleError("NonpositiveScaling")
        self.A, self.d, self.d2 = A, d, d**2

    @property
    def m(self):
        return self.A.shape[0]

    def apply(self, v):
        return self.A @ (self.d2 * (self.A.T @ v))


def pcg(op, f: Factor, p, t_max: int, tol: float):
    """krylov_solvers.py:65-105 -> (dy, residual_norms, iterations, converged)."""
    dy = np.zeros(op.m)
    r = p.copy()
    z = f.inv(r)
    gam = float(r @ z)
    if gam < 0:
        raise OracleError("Breakdown", "negative r'z")
    norms = [np.sqrt(gam)]
    if norms[0] == 0.0:
        return dy, norms, 0, True
    target = tol * norms[0]
    q = z.copy()
    its = 0
    for _ in range(t_max):
        Aq = op.apply(q)
        curv = float(q @ Aq)
        if curv <= 0:
            raise OracleError("Breakdown", f"curvature {curv:.3e}")
        a = gam / curv
        dy += a * q
        r -= a * Aq
        z = f.inv(r)
        gnew = float(r @ z)
        if gnew < 0:
            raise OracleError("Breakdown", "negative r'z")
        norms.append(float(np.sqrt(gnew)))
        its += 1
        if norms[-1] <= target:
            return dy, norms, its, True
        q = z + (gnew / gam) * q
        gam = gnew
    return dy, norms, its, False


def chebyshev(op, f: Factor, p, zeta, t_max, tol=None):
    """krylov_solvers.py:108-153 -> (dy, residual_norms, iterations, converged)."""
    if not 0.0 < zeta <= 1.0:
        raise OracleError("InvalidZeta")
    lo, hi = 2.0 / (2.0 + zeta), 2.0 / (2.0 - zeta)
    d0, c = 0.5 * (hi + lo), 0.5 * (hi - lo)
    dy = np.zeros(op.m)
    r = p.copy()
    z = f.inv(r)
    norms = [float(np.sqrt(max(r @ z, 0.0)))]
    if norms[0] == 0.0:
        return dy, norms, 0, True
    target = tol * norms[0] if tol is not None else None
    a = 0.0
    q = np.zeros(op.m)
    its = 0
    for k in range(t_max):
        if k == 0:
            q = z.copy()
            a = 1.0 / d0
        else:
            bt = (0.5 if k == 1 else 0.25) * (c * a) ** 2
            a = 1.0 / (d0 - bt / a)
            q = z + bt * q
        dy += a * q
        r -= a * op.apply(q)
        z = f.inv(r)
        norms.append(float(np.sqrt(max(r @ z, 0.0))))
        its += 1
        if target is not None and norms[-1] <= target:
            return dy, norms, its, True
    return dy, norms, its, target is None


def unpreconditioned_cg(op, p, t_max, tol):
    """krylov_solvers.py:174-204."""
    dy = np.zeros(op.m)
    r = p.copy()
    norms = [float(np.linalg.norm(r))]
    if norms[0] == 0.0:
        return dy, norms, 0, True
    target = tol * norms[0]
    gam = float(r @ r)
    q = r.copy()
    its = 0
    for _ in range(t_max):
        Aq = op.apply(q)
        curv = float(q @ Aq)
        if curv <= 0:
            raise OracleError("Breakdown", f"curvature {curv:.3e}")
        a = gam / curv
        dy += a * q
        r -= a * Aq
        gnew = float(r @ r)
        norms.append(float(np.sqrt(gnew)))
        its += 1
        if norms[-1] <= target:
            return dy, norms, its, True
        q = r + (gnew / gam) * q
        gam = gnew
    return dy, norms, its, False


def direct_solve(op, p, cap=2000):
    """krylov_solvers.py:156-171 (dense Cholesky + one refinement)."""
    import scipy.linalg
    if op.m > cap:
        raise OracleError("TooLarge")
    M = (op.A.multiply(op.d2[None, :]) @ op.A.T).toarray()
    try:
        cho = scipy.linalg.cho_factor(M, lower=True, check_finite=False)
    except scipy.linalg.LinAlgError as exc:
        raise OracleError("NotPositiveDefinite", str(exc))
    dy = scipy.linalg.cho_solve(cho, p, check_finite=False)
    dy += scipy.linalg.cho_solve(cho, p - op.apply(dy), check_finite=False)
    return dy


# ------------------------------------------------------------- correction


def compute_v(f: Factor, W: Sketch, x, s, infeas, scale):
    """correction.py:41-65 -> (v, invariant_residual)."""
    if not (np.all(x > 0) and np.all(s > 0)):
        raise OracleError("NonpositivePoint")
    u = f.pinv(infeas)
    v = np.sqrt(x * s) * W.matvec(u)
    rec = f.U @ (f.sig * (f.Vh.T @ u))
    den = scale if scale is not None else float(np.linalg.norm(infeas)) + 1.0
    if den <= 0.0:
        den = 1.0
    return v, float(np.linalg.norm(rec - infeas)) / den


# ---------------------------------------------------------- IPM step math


class Iterate:
    """ipm_core.py:70-85."""

    def __init__(self, x, y, s, r_p, r_d, mu, k=0):
        self.x, self.y, self.s, self.r_p, self.r_d, self.mu, self.k = x, y, s, r_p, r_d, mu, k

    @property
    def residual_norm(self):
        return float(math.hypot(np.linalg.norm(self.r_p), np.linalg.norm(self.r_d)))


def make_iterate(A, b, c, x, y, s, k=0):
    """ipm_core.py:88-102."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    return Iterate(x, y, s, A @ x - b, A.T @ y + s - c, float(x @ s) / x.shape[0], k)


def in_neighborhood(b, c, it, gamma, mode, r0_norm=None, mu0=None):
    """ipm_core.py:110-128."""
    if not (np.all(it.x > 0) and np.all(it.s > 0)) or it.mu <= 0:
        return False
    if np.min(it.x * it.s) < (1.0 - gamma) * it.mu - PROXIMITY_SLACK * it.mu:
        return False
    if mode == "feasible":
        return (np.linalg.norm(it.r_p) <= FEAS_TOL * (1.0 + float(np.linalg.norm(b)))
                and np.linalg.norm(it.r_d) <= FEAS_TOL * (1.0 + float(np.linalg.norm(c))))
    return it.residual_norm / max(r0_norm, 1e-300) <= it.mu / mu0 + 1e-12


def default_t_max(n, sigma, gamma, zeta):
    """ipm_core.py:176-182."""
    psi = 4.0 * math.sqrt(6.0) * (1.0 + sigma / math.sqrt(1.0 - gamma)) / (gamma * sigma)
    return max(1, math.ceil(math.log(n * psi) / math.log(1.0 / zeta)))


def build_rhs(A, it, sigma, mode):
    """ipm_core.py:196-206."""
    u = it.x - sigma * it.mu / it.s
    if mode == "feasible":
        return np.asarray(A @ u)
    u = u - (it.x / it.s) * it.r_d
    return np.asarray(A @ u) - it.r_p


def assemble_directions(A, b, it, dy, v, sigma, mode, a_scale, strict=True):
    """ipm_core.py:209-242 -> (dx, ds, cross)."""
    Atdy = np.asarray(A.T @ dy)
    ds = -Atdy if mode == "feasible" else -it.r_d - Atdy
    dx = -it.x + sigma * it.mu / it.s - (it.x / it.s) * ds - v / it.s
    if strict:
        Adx = np.asarray(A @ dx)
        row_scale = 1.0 + a_scale * float(np.linalg.norm(dx)) + float(np.linalg.norm(b))
        perr = float(np.linalg.norm(Adx)) if mode == "feasible" \
            else float(np.linalg.norm(Adx + it.r_p))
        if perr > DIRECTION_TOL * row_scale:
            raise OracleError("InvariantViolated", "primal direction row")
        derr = float(np.linalg.norm(Atdy + ds)) if mode == "feasible" \
            else float(np.linalg.norm(Atdy + ds + it.r_d))
        dscale = 1.0 + a_scale * float(np.linalg.norm(dy)) + float(np.linalg.norm(it.r_d))
        if derr > DIRECTION_TOL * dscale:
            raise OracleError("InvariantViolated", "dual direction row")
    comp = it.x * ds + it.s * dx + it.x * it.s - sigma * it.mu + v
    cscale = max(it.mu, float(np.max(np.abs(it.x * it.s))),
                 float(np.max(np.abs(it.x * ds))), float(np.max(np.abs(it.s * dx))))
    if float(np.max(np.abs(comp))) > 1e-10 * max(cscale, 1e-300):
        raise OracleError("InvariantViolated", "complementarity row")
    return dx, ds, float(dx @ ds)


def first_crossing(a, b, c):
    """ipm_core.py:245-275."""
    if np.any(c < 0):
        if np.any(c[c < 0] < -1e-12 * max(1.0, float(np.max(np.abs(c))))):
            return 0.0
        c = np.maximum(c, 0.0)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        disc = b * b - 4.0 * a * c
        real = disc >= 0
        sq = np.sqrt(np.where(real, disc, 0.0))
        qq = -0.5 * (b + np.where(b >= 0, 1.0, -1.0) * sq)
        r1 = np.where((a != 0) & real, qq / np.where(a != 0, a, 1.0), np.inf)
        r2 = np.where((qq != 0) & real, c / np.where(qq != 0, qq, 1.0), np.inf)
        r3 = np.where((a == 0) & (b < 0), -c / np.where(b < 0, b, -1.0), np.inf)
    roots = np.stack([r1, r2, r3])
    roots = np.where((roots > 0) & np.isfinite(roots), roots, np.inf)
    cand = roots.min(axis=0)
    fin = np.isfinite(cand)
    if not np.any(fin):
        return float(np.inf)
    h = 0.5 * cand[fin]
    val = a[fin] * h**2 + b[fin] * h + c[fin]
    return float(min(np.inf, np.where(val < 0, 0.0, cand[fin]).min()))


def max_alpha(A, b, c, it, dx, dy, ds, gamma, mode, r0_norm=None, mu0=None):
    """ipm_core.py:278-320 -> (alpha, probes, last_ok_iterate or None)."""
    x, s = it.x, it.s
    n = x.shape[0]
    g1 = 1.0 - gamma
    cr = dx * ds
    ln = x * ds + s * dx
    a_mu = float(cr.sum()) / n
    b_mu = float(ln.sum()) / n
    alpha = min(1.0, first_crossing(cr - g1 * a_mu, ln - g1 * b_mu, x * s - g1 * it.mu))
    alpha = min(alpha, first_crossing(np.array([a_mu]), np.array([b_mu]), np.array([it.mu])))
    if mode == "infeasible":
        ratio = it.residual_norm / max(r0_norm, 1e-300)
        alpha = min(alpha, first_crossing(np.array([a_mu / mu0]), np.array([b_mu / mu0 + ratio]),
                                          np.array([it.mu / mu0 + 1e-12 - ratio])))
    if alpha <= 0.0:
        return 0.0

    def ok(a):
        cand = make_iterate(A, b, c, x + a * dx, it.y + a * dy, s + a * ds, it.k)
        return in_neighborhood(b, c, cand, gamma, mode, r0_norm, mu0)

    if ok(alpha):
        return float(alpha)
    lo, hi = 0.0, alpha
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if ok(mid):
            lo = mid
        else:
            hi = mid
    return lo


def argmin_alpha(it, dx, ds, cross, alpha_max):
    """ipm_core.py:323-340."""
    if alpha_max <= 0.0:
        return 0.0
    lin = float(it.x @ ds + it.s @ dx)
    cands = [0.0, float(alpha_max)]
    if cross > 0.0:
        vx = -lin / (2.0 * cross)
        if 0.0 < vx < alpha_max:
            cands.append(vx)
    n = it.x.shape[0]
    return float(min(cands, key=lambda a: (n * it.mu + lin * a + cross * a * a, -a)))


# ------------------------------------------------------------ outer step


class Params:
    """The IpmParams fields the hot path reads (ipm_core.py:131-173)."""

    def __init__(self, mode="infeasible", gamma=0.5, sigma=0.5, zeta=0.5, sketch="sparse",
                 w=None, s=None, tol_cg=1e-5, tol_outer=1e-9, seed=0, max_outer=200,
                 t_max=None, solver="pcg", correction=True):
        self.mode, self.gamma, self.sigma, self.zeta = mode, gamma, sigma, zeta
        self.sketch, self.w, self.s, self.tol_cg = sketch, w, s, tol_cg
        self.tol_outer, self.seed, self.max_outer, self.t_max = tol_outer, seed, max_outer, t_max
        self.solver, self.correction = solver, correction

    @property
    def delta(self):
        return 0.1 / self.max_outer


def build_factor(A, d, prm, rng, w, s_nnz):
    """ipm_core.py:379-401 -> (Sketch, Factor, rank_retries)."""
    n = A.shape[1]
    retries = 0
    for _ in range(4):
        if w >= n:
            W = Sketch("identity", n, n, 0, 0)
        elif prm.sketch == "gaussian":
            sd = int(rng.integers(0, 2**63))
            W = Sketch("gaussian", n, w, 0, sd, dense=gaussian_sketch(n, w, sd))
        else:
            sd = int(rng.integers(0, 2**63))
            cols, vals = sparse_embedding(n, w, s_nnz, sd)
            W = Sketch("sparse_sign", n, w, s_nnz, sd, cols=cols, vals=vals)
        try:
            return W, Factor(apply_sketch(A, d, W)), retries
        except OracleError as e:
            if e.kind != "RankDeficient":
                raise
            retries += 1
            if W.kind == "identity":
                break
    raise OracleError("RankDeficient", f"after {retries} resketches")


def ipm_step(A, b, c, it, prm, rng, r0_norm=None, mu0=None, a_scale=None, trace_hook=None):
    """ipm_core.py:404-585 (pcg solver, correction on) -> (new iterate, record dict)."""
    mode = prm.mode
    if not in_neighborhood(b, c, it, prm.gamma, mode, r0_norm, mu0):
        raise OracleError("NeighborhoodViolated", f"iterate {it.k}")
    if a_scale is None:
        a_scale = math.sqrt(float((A.data**2).sum()))
    ratio = it.x / it.s
    clipped = np.clip(ratio, RATIO_FLOOR, RATIO_CAP)
    clip_count = int(np.count_nonzero(clipped != ratio))
    d = np.sqrt(clipped)
    op = NormalOp(A, d)
    p = build_rhs(A, it, prm.sigma, mode)
    p_norm = float(np.linalg.norm(p))
    t_base = prm.t_max if prm.t_max is not None else default_t_max(A.shape[1], prm.sigma,
                                                                     prm.gamma, prm.zeta)
    tol_eff = prm.tol_cg
    if not prm.correction or prm.solver == "unpreconditioned":      # ipm_core.py:436-448
        if mode == "infeasible":
            budget = 0.05 * (it.mu / mu0) * r0_norm
        else:
            budget = 0.05 * FEAS_TOL * (1.0 + float(np.linalg.norm(b))) / max(prm.max_outer, 1)
        tol_eff = max(min(prm.tol_cg, budget / max(p_norm, 1e-300)), 1e-14)
        t_deep = math.ceil(math.log(1.0 / tol_eff) / math.log(1.0 / prm.zeta)) + 2
        t_base = max(t_base, t_deep)
    W = f = None
    seed = None
    w = 0
    rank_retries = v_retries = inner_total = 0
    v = infeas = None
    vnorm, slack = 0.0, float("nan")
    if prm.solver == "direct":                                         # ipm_core.py:450-453
        dy = direct_solve(op, p)
        norms, its = [p_norm, float(np.linalg.norm(op.apply(dy) - p))], 0
    elif prm.solver == "unpreconditioned":                             # ipm_core.py:454-456
        dy, norms, its, conv = unpreconditioned_cg(op, p, max(1000, 20 * A.shape[0]), tol_eff)
        inner_total = its
    else:
        w, s_nnz = auto_sketch_dims(A.shape[0], A.shape[1], prm.delta)
        if prm.w is not None:
            w = prm.w
        if prm.s is not None:
            s_nnz = prm.s
        best = chosen = None
        sched = [(True, t_base), (False, 2 * t_base)] + [(True, 2 * t_base)] * 3
        for fresh, t_eff in sched:
            if fresh or W is None:
                W, f, rr = build_factor(A, d, prm, rng, w, s_nnz)
                rank_retries += rr
                seed = W.seed
            if prm.solver == "chebyshev":
                dy, norms, its, conv = chebyshev(op, f, p, prm.zeta, t_eff,
                                                 None if prm.correction else tol_eff)
            else:
                dy, norms, its, conv = pcg(op, f, p, t_eff, tol_eff)
            if trace_hook is not None:
                trace_hook(W, f, dy, norms)
            inner_total += its
            if not prm.correction:
                chosen = (dy, norms, its, None, 0.0, float("nan"), None)
                break
            infeas = op.apply(dy) - p
            scale = float(np.linalg.norm(infeas)) + p_norm
            v, inv_res = compute_v(f, W, it.x, it.s, infeas, scale if scale > 0 else 1.0)
            vnorm = float(np.linalg.norm(v))
            slack = float(np.sqrt(3.0 * A.shape[1] * it.mu) * norms[-1] - vnorm)
            cand = (dy, norms, its, v, vnorm, slack, infeas)
            if vnorm <= prm.gamma * prm.sigma * it.mu / 4.0:
                chosen = cand
                break
            v_retries += 1
            if best is None or vnorm < best[4]:
                best = cand
        if chosen is None:
            chosen = best
        dy, norms, its, v, vnorm, slack, infeas = chosen

    v_inv = float("nan")
    if v is not None:
        scale = float(np.linalg.norm(infeas)) + p_norm
        v_inv = float(np.linalg.norm(np.asarray(A @ (v / it.s)) - infeas)) / max(scale, 1e-300)
        if v_inv > V_INVARIANT_TOL:
            raise OracleError("InvariantViolated", f"correction invariant {v_inv:.3e}")
    else:
        v = np.zeros(A.shape[1])
    strict = prm.solver == "direct" or v_inv == v_inv
    dx, ds, cross = assemble_directions(A, b, it, dy, v, prm.sigma, mode, a_scale, strict)
    at = max_alpha(A, b, c, it, dx, dy, ds, prm.gamma, mode, r0_norm, mu0)
    ab = argmin_alpha(it, dx, ds, cross, at)
    new = make_iterate(A, b, c, it.x + ab * dx, it.y + ab * dy, it.s + ab * ds, it.k + 1)

    n = A.shape[1]
    v_bar = float(v.sum()) / n
    pred_lin = (1.0 - ab * (1.0 - prm.sigma)) * it.mu - ab * v_bar
    pred_quad = pred_lin + ab**2 * cross / n
    mu_scale = max(it.mu, abs(pred_quad), 1e-300)
    mu_err = abs(new.mu - pred_quad) / mu_scale
    if mu_err > MU_IDENTITY_TOL:
        raise OracleError("InvariantViolated", "mu identity")
    if mode == "feasible" and abs(new.mu - pred_lin) > MU_IDENTITY_TOL * mu_scale:
        raise OracleError("InvariantViolated", "linear mu identity")
    if new.mu > it.mu * (1.0 + 1e-12):
        raise OracleError("InvariantViolated", "mu increased")
    v_ok = v_inv == v_inv and vnorm <= prm.gamma * prm.sigma * it.mu / 4.0
    if mode == "feasible" and v_ok:
        if new.mu > (1.0 - 0.5 * ab * (1.0 - 1.25 * prm.sigma)) * it.mu * (1.0 + 1e-10):
            raise OracleError("InvariantViolated", "mu decrease bound")
    if mode == "feasible":
        if (np.linalg.norm(new.r_p) > FEAS_TOL * (1.0 + float(np.linalg.norm(b)))
                or np.linalg.norm(new.r_d) > FEAS_TOL * (1.0 + float(np.linalg.norm(c)))):
            raise OracleError("InvariantViolated", "residual drift")
    if not in_neighborhood(b, c, new, prm.gamma, mode, r0_norm, mu0):
        raise OracleError("NeighborhoodViolated", f"step {it.k}")
    rec = dict(
        k=it.k, mu=float(it.mu), mu_after=float(new.mu), alpha_tilde=float(at),
        alpha_bar=float(ab), inner_iterations=its, inner_iterations_total=inner_total,
        f_norm0=float(norms[0]), f_norm=float(norms[-1]), v_norm=vnorm, v_bar=v_bar,
        v_invariant_rel=v_inv, v_norm_slack=slack, v_ok=bool(v_ok), v_retries=v_retries,
        rank_retries=rank_retries, sketch_w=w if prm.solver in ("pcg", "chebyshev") else 0,
        sketch_seed=seed,
        residual_ratio=float(new.residual_norm / max(r0_norm, 1e-300))
        if r0_norm is not None else float("nan"),
        mu_identity_error=float(mu_err), clip_count=clip_count,
        inner_residual_norms=[float(r) for r in norms],
    )
    return new, rec


def solve(A, b, c, start: Iterate, prm: Params, max_steps=None, on_step=None):
    """ipm_core.py:665-734 with a given start -> dict summary (+ records).

    on_step(k, it, rng_state) is called before each outer step (lock-step
    harness snapshots)."""
    rng = philox(prm.seed)
    mu0 = start.mu
    r0 = max(start.residual_norm, 1e-300)
    eps = prm.tol_outer * max(1.0, mu0)
    if prm.mode == "feasible" and not in_neighborhood(b, c, start, prm.gamma, "feasible"):
        raise OracleError("NeighborhoodViolated", "start")
    gamma = prm.gamma
    if prm.mode == "infeasible" and not in_neighborhood(b, c, start, prm.gamma, "infeasible",
                                                        r0, mu0):
        th = float(np.min(start.x * start.s) / mu0)
        gamma = min(1.0 - 1e-12, max(prm.gamma, 1.0 - 0.999 * th))
    run = Params(**{k: getattr(prm, k) for k in vars(prm)})
    run.gamma = gamma
    a_scale = math.sqrt(float((A.data**2).sum()))
    it = start
    recs = []
    while it.mu > eps:
        if len(recs) >= prm.max_outer or (max_steps is not None and len(recs) >= max_steps):
            break
        if on_step is not None:
            on_step(len(recs), it, rng.bit_generator.state)
        it, rec = ipm_step(A, b, c, it, run, rng, r0, mu0, a_scale)
        recs.append(rec)
    return dict(
        converged=bool(it.mu <= eps), outer=len(recs),
        sum_inner=sum(r["inner_iterations_total"] for r in recs),
        max_inner=max((r["inner_iterations"] for r in recs), default=0),
        mu0=float(mu0), mu_final=float(it.mu), epsilon=float(eps),
        objective=float(c @ it.x), dual_objective=float(b @ it.y),
        mu_trace=[float(mu0)] + [r["mu_after"] for r in recs],
        gamma_effective=gamma, steps=recs, x=it.x, y=it.y, s=it.s,
    )
