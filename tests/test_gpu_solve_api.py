"""Solver API behaviour on the device, mirroring the reference's own solve /
feasible-start tests (reference tests/test_ipm_core.py:419-545): trivial LPs in
both modes, determinism, monotone mu, MaxIterations with its partial report,
unbounded and infeasible detection, all inner solvers reaching the LP optimum
(checked with scipy's HiGHS as an independent oracle), gamma widening,
circulation pairs, the mu identity replayed from the records, feasible-start
membership."""

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.optimize import linprog

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def IC():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_08722_b200 import ipm_core
    return ipm_core


def _lp(A, b, c, name="lp"):
    from paper_2209_08722_b200.lp_model import make_lp
    return make_lp(sp.csr_matrix(np.asarray(A, dtype=np.float64)), b, c, name=name)


def _feasible(m, n, density, seed):
    from paper_2209_08722_b200.problems import random_feasible_dense
    return _lp(*random_feasible_dense(m, n, density, seed))


def _optimum(lp):
    r = linprog(lp.c, A_eq=lp.A.toarray(), b_eq=lp.b, bounds=(0, None), method="highs")
    assert r.status == 0
    return r.fun


def test_trivial_lp_both_modes(IC):
    lp = _lp([[1.0]], np.array([1.0]), np.array([1.0]), "unit")
    for mode in ("infeasible", "feasible"):
        rep = IC.solve(lp, params=IC.IpmParams(mode=mode))
        assert rep.converged
        assert abs(rep.x[0] - 1.0) <= 1e-6 and abs(rep.gap) <= 1e-8


def test_deterministic_and_monotone(IC):
    lp = _feasible(5, 20, 0.3, 7)
    a = IC.solve(lp, params=IC.IpmParams(seed=3))
    b = IC.solve(lp, params=IC.IpmParams(seed=3))
    assert np.array_equal(a.x, b.x) and a.mu_trace == b.mu_trace
    assert [r.sketch_seed for r in a.steps] == [r.sketch_seed for r in b.steps]
    t = a.mu_trace
    assert all(t[i + 1] <= t[i] * (1 + 1e-12) for i in range(len(t) - 1))
    assert a.mu_final <= a.epsilon


def test_max_iterations_carries_partial_report(IC):
    from paper_2209_08722_b200.errors import MaxIterations
    lp = _feasible(5, 20, 0.3, 7)
    with pytest.raises(MaxIterations) as exc:
        IC.solve(lp, params=IC.IpmParams(max_outer=2))
    rep = exc.value.report
    assert rep is not None and not rep.converged
    assert rep.outer == 2 and len(rep.steps) == 2 and rep.mu_final > rep.epsilon


def test_unbounded_detection(IC):
    from paper_2209_08722_b200.errors import MaxIterations, Unbounded
    lp = _lp([[1.0, -1.0]], np.array([1.0]), np.array([-1.0, 0.0]), "ray")
    with pytest.raises(Unbounded):
        IC.feasible_start(lp)
    with pytest.raises((MaxIterations, Unbounded)):
        IC.solve(lp, params=IC.IpmParams(mode="infeasible", max_outer=300))


def test_infeasible_instance_detected(IC):
    from paper_2209_08722_b200.errors import Infeasible
    from paper_2209_08722_b200.problems import random_dense
    lp = _lp(*random_dense(20, 400, 0.3, 1))
    with pytest.raises(Infeasible):
        IC.phase1_point(lp)


def test_objective_matches_highs_infeasible_mode(IC):
    lp = _feasible(20, 400, 0.3, 1)
    rep = IC.solve(lp, params=IC.IpmParams(mode="infeasible"))
    ref = _optimum(lp)
    assert rep.converged and abs(rep.objective - ref) <= 1e-6 * max(1.0, abs(ref))


@pytest.mark.parametrize("solver", ["pcg", "chebyshev", "direct", "unpreconditioned"])
def test_all_solvers_agree(IC, solver):
    lp = _feasible(5, 30, 0.4, 2)
    rep = IC.solve(lp, params=IC.IpmParams(solver=solver, seed=0))
    ref = _optimum(lp)
    assert rep.converged and abs(rep.objective - ref) <= 1e-6 * max(1.0, abs(ref))


def test_gamma_widens_for_off_center_start(IC):
    lp = _feasible(4, 12, 0.5, 3)
    x0 = np.ones(12)
    x0[0] = 1e-4
    start = IC.make_iterate(IC._to_device_lp(lp, None), x0, np.ones(4), np.ones(12))
    theta0 = float(start.min_xs / start.mu)
    expected = max(0.5, 1.0 - 0.999 * theta0)
    rep = IC.solve(lp, start=start, params=IC.IpmParams(mode="infeasible", max_outer=400))
    assert rep.converged and abs(rep.gamma_effective - expected) <= 1e-15


def test_circulation_pair_stays_bounded(IC):
    lp = _lp([[1.0, -1.0, 1.0]], np.array([1.0]), np.array([0.0, 0.0, 1.0]), "circ")
    rep = IC.solve(lp, params=IC.IpmParams(mode="infeasible"))
    assert rep.converged and abs(rep.objective) <= 1e-6 and float(np.max(rep.x)) < 1e3


def test_mu_identity_recomputable_from_records(IC):
    lp = _feasible(5, 20, 0.3, 7)
    params = IC.IpmParams(mode="feasible", seed=0)
    rep = IC.solve(lp, params=params)
    for rec in rep.steps:
        pred = (1.0 - rec.alpha_bar * (1.0 - params.sigma)) * rec.mu - rec.alpha_bar * rec.v_bar
        assert abs(rec.mu_after - pred) <= 1e-9 * max(rec.mu, 1e-300)
        assert rec.mu_identity_error <= 1e-10


def test_feasible_start_membership(IC):
    lp = _feasible(5, 20, 0.3, 7)
    dlp = IC._to_device_lp(lp, None)
    start = IC.feasible_start(lp)
    assert start.k == 0 and start.mu <= 1.0 + 1e-12
    assert IC.in_neighborhood(dlp, start, 0.5, "feasible")
    lp2 = _feasible(4, 12, 0.5, 3)
    st2 = IC.feasible_start(lp2, IC.IpmParams(mode="feasible", gamma=0.3))
    assert IC.in_neighborhood(IC._to_device_lp(lp2, None), st2, 0.3, "feasible")


def test_diag_cond_matches_reference(IC):
    """diag_cond diagnostics (reference ipm_core.py:576-584): spectrum bounds of
    the preconditioned normal matrix and cond(AD)^2 per step, against the
    reference's dense-SVD values (tests/golden/diag_traces.json)."""
    import json
    import os
    from conftest import GOLDEN
    from paper_2209_08722_b200.lp_model import LinearProgram
    from paper_2209_08722_b200.problems import wide_dense_lp
    with open(os.path.join(GOLDEN, "diag_traces.json")) as f:
        gold = json.load(f)
    lpd = wide_dense_lp(40, 3000, 5)
    lp = LinearProgram(sp.csr_matrix(lpd.A), lpd.b, lpd.c)
    st = IC.make_iterate(IC._to_device_lp(lp, None), lpd.x0, lpd.y0, lpd.s0)
    rep = IC.solve(lp, st, IC.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5,
                                        w=160, s=4, tol_outer=1e-6, seed=3, diag_cond=True))
    assert rep.outer == gold["outer"]
    for rec, g in zip(rep.steps, gold["steps"]):
        for k in ("spectrum_lo", "spectrum_hi", "kappa_sk"):
            assert abs(getattr(rec, k) - g[k]) <= 1e-7 * abs(g[k]), (k, getattr(rec, k), g[k])
        # cond(AD)^2 from the explicit Gram (the reference squares SVD values): looser
        assert abs(rec.kappa_stan - g["kappa_stan"]) <= 1e-4 * g["kappa_stan"]


def test_diag_cond_cap(IC):
    from paper_2209_08722_b200.errors import TooLargeForDiagnostic
    g = np.random.Generator(np.random.Philox(1))
    m, n = 70, 1_000_000          # m * n above the reference's 2^26 cap
    A = g.standard_normal((m, n))
    lp = _lp(A, A @ (g.random(n) + 0.5), A.T @ g.standard_normal(m) + g.random(n) + 0.5)
    with pytest.raises(TooLargeForDiagnostic):
        IC.solve(lp, params=IC.IpmParams(mode="infeasible", diag_cond=True, max_outer=1))
