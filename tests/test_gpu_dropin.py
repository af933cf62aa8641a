"""The drop-in boundary on the device: the reference's own CLI
(skipm.cli.main, cli.py:465-536) routed to the B200 solve by the one-line
patch INTEGRATION.md shows (cli.py binds `solve` by name at import,
cli.py:30), with the reference's exit codes (cli.py:49-52) for a converged
run, an exhausted outer budget (MaxIterations) and a device failure, and the
reference's exception classes caught from device-detected failures."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

skipm = pytest.importorskip("skipm")


@pytest.fixture()
def problem_dir(tmp_path):
    lp = skipm.random_feasible_lp(20, 200, 0.5, 3)
    return skipm.save_matrix_market(lp, str(tmp_path / "prob"))


@pytest.fixture()
def device_cli(monkeypatch):
    import skipm.cli as cli

    import paper_2209_08722_b200 as skb
    calls = []

    def device_solve(lp, start=None, params=None):
        calls.append(params)
        return skb.solve(lp, start, params)

    monkeypatch.setattr(cli, "solve", device_solve)
    return cli, calls


def test_cli_solve_on_device_matches_reference_trace(problem_dir, device_cli, tmp_path,
                                                     golden_dir):
    cli, calls = device_cli
    out = tmp_path / "report.json"
    rc = cli.main(["solve", problem_dir, "--mode", "feasible", "--gamma", "0.5", "--sigma", "0.5",
                   "--tol-outer", "1e-6", "--seed", "2", "--out", str(out), "--no-timestamp"])
    assert rc == cli.EXIT_OK and len(calls) == 1
    assert isinstance(calls[0], skipm.IpmParams)
    rep = json.load(open(out))  # already validated against REPORT_SCHEMA by the CLI
    with open(os.path.join(golden_dir, "start_traces.json")) as f:
        ref = json.load(f)["solve"]  # the reference's own solve of this problem
    assert rep["converged"] and rep["outer"] == ref["outer"]
    assert rep["inner_iterations"] == [s["inner_iterations"] for s in ref["steps"]]
    assert abs(rep["objective"] - ref["objective"]) <= 1e-8 * abs(ref["objective"])
    mu = np.abs(np.array(rep["mu_trace"]) - ref["mu_trace"]) / np.array(ref["mu_trace"])
    print(f"cli on device: outer {rep['outer']}, max mu rel dev {mu.max():.2e}")
    assert mu.max() <= 1e-9


def test_cli_max_iterations_exit_code(problem_dir, device_cli, capsys):
    cli, calls = device_cli
    rc = cli.main(["solve", problem_dir, "--mode", "infeasible", "--max-outer", "2",
                   "--tol-outer", "1e-9", "--no-timestamp", "--out", os.devnull])
    assert rc == cli.EXIT_NUMERIC and calls
    assert "MaxIterations" in capsys.readouterr().err


def test_cli_device_failure_exit_code(problem_dir, device_cli, monkeypatch, capsys):
    cli, _ = device_cli
    from paper_2209_08722_b200 import _lib, ipm_core

    def failing_step(*a, **k):
        raise _lib.SkbError("skb_normal_apply", -4)

    monkeypatch.setattr(ipm_core, "ipm_step", failing_step)
    rc = cli.main(["solve", problem_dir, "--mode", "infeasible", "--no-timestamp",
                   "--out", os.devnull])
    assert rc == cli.EXIT_NUMERIC
    assert "SkbError" in capsys.readouterr().err


def test_reference_except_clause_catches_device_rank_deficiency():
    """RankDeficient iff sigma_min/sigma_max(ADW) < 1e-12 (preconditioning.py:47-50),
    decided on the device from the factor, caught by the reference's class."""
    import torch

    from paper_2209_08722_b200 import preconditioning as PC
    from paper_2209_08722_b200.kernels import DeviceMatrix
    from paper_2209_08722_b200.runtime import F64, lda_for
    m, w = 64, 256
    rng = np.random.Generator(np.random.Philox(5))

    def device_x(adw):
        cols = torch.zeros((w, lda_for(m)), dtype=F64, device="cuda")
        cols[:, :m] = torch.from_numpy(np.ascontiguousarray(adw.T)).cuda()
        return DeviceMatrix(cols, m)

    G = rng.standard_normal((m, w))
    zero = G.copy()
    zero[7] = 0.0  # rank m - 1
    with pytest.raises(skipm.errors.RankDeficient):
        PC.build_preconditioner(device_x(zero))
    # graded rows: sigma ratio 1.31e-12 (full rank for the reference) -> accepted;
    # the Frobenius lower bound (7.5e-13) is below 1e-12 here, so the converged
    # power iterations decide
    graded = (10.0 ** np.linspace(0, -11.8, m))[:, None] * G
    sv = np.linalg.svd(graded, compute_uv=False)
    ratio = sv[-1] / sv[0]
    assert ratio > 1e-12
    f = PC.build_preconditioner(device_x(graded))
    lo, hi = PC.sigma_ratio_bounds(f, exact=True)
    print(f"graded: svd ratio {ratio:.4e}, device bounds [{lo:.4e}, {hi:.4e}]")
    # kappa(ADW) ~ 8e11: the factor's singular values carry ~u*kappa relative error
    assert lo <= ratio * (1 + 1e-2) and hi >= ratio * (1 - 1e-2)
    assert abs(hi - ratio) <= 1e-2 * ratio  # the converged estimate
    # one more decade: ratio below 1e-12 -> RankDeficient like the reference
    steep = (10.0 ** np.linspace(0, -12.5, m))[:, None] * G
    sv = np.linalg.svd(steep, compute_uv=False)
    assert sv[-1] / sv[0] < 1e-12
    with pytest.raises(skipm.errors.RankDeficient):
        PC.build_preconditioner(device_x(steep))
