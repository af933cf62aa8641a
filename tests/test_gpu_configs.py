"""Parity at the BASELINE configurations' own problem sizes, against traces
recorded from the LIVE reference (tests/golden/make_golden_configs.py; the
reference's SolveReport of the first K outer steps, or of the whole solve).

The LP is regenerated on the box host with the seeded generator of SURVEY.md
§8(d) (paper_2209_08722_b200/problems.py: the same numpy Philox draw order
the golden script used), uploaded, and solved on the device with the same
IpmParams. Gates (BASELINE.json north_star, reference ipm_core.py:404-585):
sketch seeds, inner iteration counts, v_retries and rank_retries identical;
mu_after, alpha_tilde and alpha_bar within 1e-9 relative; PCG residual norms
within 1e-9 * f_norm0 (1e-8 * f_norm0 for the ill-conditioned c5 generator,
whose measured floor is 3.2e-9 * f_norm0 for every factorization, SURVEY.md
§8(c)); the objective of a full solve within 1e-8 relative. Every test
prints the largest deviation it measured.

  c2         1000 x 1e6 dense (8 GB), w=4000, s=4 and s=1: 3 steps each
  m1000      1000 x 1e5 dense, w=4000, s=4: the whole solve to mu < 1e-8
  m2000      2000 x 1e5 dense, w=8000, s=4: 6 steps (the warp-pair K4 kernel)
  sparse1e4  1e4 x 2e5 CSC (5 nnz/col), w=4e4, s=4: 3 steps (L2 CSC sketch,
             INT8-emulated factor GEMMs)
  c4         c4 itself: 1e4 x 2e7 CSC (1e8 nnz), w=4e4, s=4: 2 steps (the CSC sketch
             and the INT8-emulated factor at full size; the reference takes 436 s a step)
  c5m1000    ill-conditioned 1000 x 2e4, Gaussian w=4000, sigma=0.3: 6 steps
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
CASES = ["c2", "m1000", "m2000", "sparse1e4", "c4", "c5m1000"]


def _load(case):
    path = os.path.join(GOLDEN, f"cfg_{case}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        return json.load(f)


def _host_lp(gen):
    from paper_2209_08722_b200.problems import (ill_conditioned_lp, sparse_wide_lp,
                                                wide_dense_lp)
    kind, m, n, seed = gen
    if kind == "dense":
        return wide_dense_lp(m, n, seed)
    if kind == "ill":
        return ill_conditioned_lp(m, n, seed)
    return sparse_wide_lp(m, n, 5, seed)


def _rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


def compare_steps(rep, gold, rn_tol=1e-9, tag=""):
    """Step-by-step comparison; returns the measured maxima (also printed)."""
    assert rep.outer == gold["outer"], (rep.outer, gold["outer"])
    steps = gold["steps"]
    assert [r.sketch_seed for r in rep.steps] == [s["sketch_seed"] for s in steps]
    assert [r.inner_iterations for r in rep.steps] == [s["inner_iterations"] for s in steps]
    assert [r.v_retries for r in rep.steps] == [s["v_retries"] for s in steps]
    assert [r.rank_retries for r in rep.steps] == [s["rank_retries"] for s in steps]
    assert [r.inner_iterations_total for r in rep.steps] == \
        [s["inner_iterations_total"] for s in steps]
    dev = {"mu": 0.0, "alpha_tilde": 0.0, "alpha_bar": 0.0, "residual/f0": 0.0}
    for r, s in zip(rep.steps, steps):
        dev["mu"] = max(dev["mu"], float(_rel(r.mu_after, s["mu_after"])))
        dev["alpha_tilde"] = max(dev["alpha_tilde"], float(_rel(r.alpha_tilde, s["alpha_tilde"])))
        dev["alpha_bar"] = max(dev["alpha_bar"], float(_rel(r.alpha_bar, s["alpha_bar"])))
        a, b = np.array(r.inner_residual_norms), np.array(s["inner_residual_norms"])
        assert a.shape == b.shape
        dev["residual/f0"] = max(dev["residual/f0"],
                                 float(np.max(np.abs(a - b)) / s["f_norm0"]))
    print(f"[{tag}] outer {rep.outer}: max deviations " +
          ", ".join(f"{k} {v:.2e}" for k, v in dev.items()))
    assert dev["mu"] <= 1e-9 and dev["alpha_tilde"] <= 1e-9 and dev["alpha_bar"] <= 1e-9, dev
    assert dev["residual/f0"] <= rn_tol, dev
    return dev


def _solve(lpd, dlp, gold_case, key, s_nnz):
    from paper_2209_08722_b200 import ipm_core as IC
    from paper_2209_08722_b200.errors import MaxIterations
    kw = dict(mode="feasible", gamma=gold_case["gamma_run"], sigma=gold_case["sigma"],
              sketch=gold_case["sketch"], w=gold_case["w"], tol_outer=gold_case["tol_outer"],
              seed=gold_case["seed"])
    if gold_case["sketch"] == "sparse":
        kw["s"] = s_nnz
    if gold_case["steps_limit"] is not None:
        kw["max_outer"] = gold_case["steps_limit"]
    start = IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0)
    try:
        return IC.solve(dlp, start, IC.IpmParams(**kw))
    except MaxIterations as e:
        assert gold_case["steps_limit"] is not None
        return e.report


@pytest.mark.parametrize("case", CASES)
def test_config_trajectory_vs_live_reference(case):
    import torch

    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    g = _load(case)
    lpd = _host_lp(g["gen"])
    dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c, name=lpd.name))
    del lpd.A
    keys = [k for k in ("s4", "s1", "gaussian") if k in g]
    assert keys
    for key in keys:
        gold = g[key]
        s_nnz = int(key[1:]) if key.startswith("s") else 0
        rep = _solve(lpd, dlp, g, key, s_nnz)
        rn_tol = 1e-8 if g["gen"][0] == "ill" else 1e-9
        compare_steps(rep, gold, rn_tol=rn_tol, tag=f"{case}/{key}")
        if gold["converged"]:
            assert rep.converged
            assert float(_rel(rep.objective, gold["objective"])) <= 1e-8
            print(f"[{case}/{key}] objective rel dev "
                  f"{float(_rel(rep.objective, gold['objective'])):.2e}")
        y_head = rep.y[:8]
        assert np.allclose(y_head, gold["y_head"], rtol=1e-7, atol=1e-9 * gold["y_norm"])
    del dlp
    torch.cuda.empty_cache()
