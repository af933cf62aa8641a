"""Golden traces of the LIVE reference at the BASELINE configs' own problem sizes.

Run in the build container (where /root/reference exists), one case at a time
(c2 needs ~30 GB of host memory and ~2-3 min per outer step on 8 cores):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden_configs.py c2 m1000 ...

Each case writes tests/golden/cfg_<case>.json: the reference's SolveReport
(StepRecords: sketch seeds, inner/v/rank retries, mu/alpha, PCG residual
traces) for the first K outer steps (K = all for the full solves), plus the
wall time per outer step of the reference on this host.
The GPU tests (tests/test_gpu_configs.py) regenerate the same A on the box
host from the seeded generator (paper_2209_08722_b200/problems.py, the draw
order of SURVEY.md §8(d)), solve on the device, and compare step by step.

Cases (SURVEY.md §8(d) generators; gamma widened as in App. C):
  c2        wide_dense_lp(1000, 1_000_000, 0), w=4000, s=4 and s=1, 3 steps each
  m1000     wide_dense_lp(1000, 100_000, 1),   w=4000, s=4, full solve to mu<1e-8
  m2000     wide_dense_lp(2000, 100_000, 2),   w=8000, s=4, 6 steps (warp-pair K4)
  sparse1e4 sparse_wide_lp(10_000, 200_000, 5, 3), w=40_000, s=4, 3 steps
            (L2 CSC sketch, INT8-emulated factor GEMMs at m=1e4)
  c4        sparse_wide_lp(10_000, 20_000_000, 5, 4) -- c4 itself, 1e8 nnz -- w=40_000, s=4,
            2 steps (the reference's gesdd of the 1e4 x 4e4 sketch dominates its step)
  c5m1000   ill_conditioned_lp(1000, 20_000, 4), Gaussian w=4000, sigma=0.3, 6 steps
            (scipy's sparse x dense AD @ W is single-threaded: ~1 min per sketch here)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

import scipy.sparse as sp  # noqa: E402

import skipm  # noqa: E402
from skipm import ipm_core, krylov_solvers, preconditioning, sketching  # noqa: E402

from paper_2209_08722_b200.problems import (ill_conditioned_lp, sparse_wide_lp,  # noqa: E402
                                            wide_dense_lp)

CASES = {
    "c2": dict(gen=("dense", 1000, 1_000_000, 0), w=4000, sketch="sparse", s=(4, 1),
               sigma=0.5, tol=1e-8, steps=3, seed=0),
    "m1000": dict(gen=("dense", 1000, 100_000, 1), w=4000, sketch="sparse", s=(4,),
                  sigma=0.5, tol=1e-8, steps=None, seed=1),
    "m2000": dict(gen=("dense", 2000, 100_000, 2), w=8000, sketch="sparse", s=(4,),
                  sigma=0.5, tol=1e-8, steps=6, seed=2),
    "sparse1e4": dict(gen=("sparse", 10_000, 200_000, 3), w=40_000, sketch="sparse", s=(4,),
                      sigma=0.5, tol=1e-8, steps=3, seed=3),
    "c5m1000": dict(gen=("ill", 1000, 20_000, 4), w=4000, sketch="gaussian", s=(0,),
                    sigma=0.3, tol=1e-8, steps=6, seed=4),
    "c4": dict(gen=("sparse", 10_000, 20_000_000, 4), w=40_000, sketch="sparse", s=(4,),
               sigma=0.5, tol=1e-8, steps=2, seed=4),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dense_csr(A: np.ndarray) -> sp.csr_matrix:
    """CSR of a dense row-major A sharing its buffer (no COO transient; row-major
    dense IS the CSR data order). Index dtype int32 while nnz < 2^31."""
    m, n = A.shape
    idx_t = np.int32 if m * n < 2**31 else np.int64
    indices = np.tile(np.arange(n, dtype=idx_t), m)
    indptr = np.arange(0, m * n + 1, n, dtype=idx_t if m * n < 2**31 else np.int64)
    out = sp.csr_matrix((A.reshape(-1), indices, indptr), shape=(m, n), copy=False)
    out.has_sorted_indices = True
    return out


def make(gen):
    kind, m, n, seed = gen
    if kind == "dense":
        lpd = wide_dense_lp(m, n, seed)
        A = dense_csr(lpd.A)
    elif kind == "ill":
        lpd = ill_conditioned_lp(m, n, seed)
        A = dense_csr(lpd.A)
    else:
        lpd = sparse_wide_lp(m, n, 5, seed)
        A = lpd.A.tocsr()
        A.sort_indices()
    lp = skipm.make_lp(A, lpd.b, lpd.c, name=lpd.name)
    return lpd, lp


def cpu_kernels_c2(lpd, lp):
    """Reference functions at full c2 size on this host."""
    out = {"host_cores": os.cpu_count()}
    g = np.random.Generator(np.random.Philox(5))
    d = np.sqrt(g.uniform(0.5, 1.5, lp.n) / g.uniform(0.5, 1.5, lp.n))
    op = krylov_solvers.NormalOperator(lp.A, d)
    z = g.standard_normal(lp.m)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        op.apply(z)
        ts.append(time.perf_counter() - t0)
    out["normal_apply_s"] = min(ts)
    for s_nnz in (1, 4):
        W = sketching.build_sparse_embedding(lp.n, 4000, s_nnz, 11)
        t0 = time.perf_counter()
        X = sketching.apply_sketch(lp.A, d, W)
        out[f"apply_sketch_s{s_nnz}_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    preconditioning.build_preconditioner(X, sketch_tag=W.tag) if "sketch_tag" in \
        preconditioning.build_preconditioner.__code__.co_varnames else \
        preconditioning.build_preconditioner(X)
    out["build_preconditioner_s"] = time.perf_counter() - t0
    return out


def run_case(name):
    cfg = CASES[name]
    t0 = time.perf_counter()
    lpd, lp = make(cfg["gen"])
    res = {"case": name, "gen": list(cfg["gen"]), "w": cfg["w"], "sketch": cfg["sketch"],
           "sigma": cfg["sigma"], "tol_outer": cfg["tol"], "steps_limit": cfg["steps"],
           "seed": cfg["seed"], "gamma_run": lpd.gamma_run(0.1),
           "b_sha256": sha(lpd.b), "c_sha256": sha(lpd.c), "gen_seconds": 0.0,
           "host_cores": os.cpu_count()}
    res["gen_seconds"] = time.perf_counter() - t0
    print(f"[{name}] generated m={lp.m} n={lp.n} nnz={lp.A.nnz} in {res['gen_seconds']:.1f}s",
          flush=True)
    for s_nnz in cfg["s"]:
        start = ipm_core.make_iterate(lp, lpd.x0, lpd.y0, lpd.s0)
        kw = dict(mode="feasible", gamma=res["gamma_run"], sigma=cfg["sigma"],
                  sketch=cfg["sketch"], w=cfg["w"], tol_outer=cfg["tol"], seed=cfg["seed"])
        if cfg["sketch"] == "sparse":
            kw["s"] = s_nnz
        if cfg["steps"] is not None:
            kw["max_outer"] = cfg["steps"]
        prm = ipm_core.IpmParams(**kw)
        t1 = time.perf_counter()
        try:
            rep = ipm_core.solve(lp, start, prm)
        except skipm.MaxIterations as e:
            rep = e.report
        wall = time.perf_counter() - t1
        d = rep.to_dict()
        d.pop("params")
        d["x_sha256"] = sha(rep.x)
        d["x_head"] = rep.x[:8].tolist()
        d["y_head"] = rep.y[:8].tolist()
        d["y_norm"] = float(np.linalg.norm(rep.y))
        d["wall_seconds_solve"] = wall
        d["seconds_per_outer"] = wall / max(rep.outer, 1)
        key = f"s{s_nnz}" if cfg["sketch"] == "sparse" else "gaussian"
        res[key] = d
        print(f"[{name}] {key}: outer {rep.outer} inner {rep.sum_inner} conv {rep.converged} "
              f"mu {rep.mu_final:.4e} obj {rep.objective!r} ({wall:.0f}s, "
              f"{wall / max(rep.outer, 1):.1f}s/outer)", flush=True)
        with open(os.path.join(HERE, f"cfg_{name}.json"), "w") as f:
            json.dump(res, f)
    if name == "c2":
        res["cpu_kernels"] = cpu_kernels_c2(lpd, lp)
        print(f"[{name}] cpu kernels {res['cpu_kernels']}", flush=True)
    with open(os.path.join(HERE, f"cfg_{name}.json"), "w") as f:
        json.dump(res, f)


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        run_case(name)
