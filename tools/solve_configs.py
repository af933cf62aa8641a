"""Full-size IPM time-to-solve for BASELINE configs c3, c4, c5 on ONE B200
(synthetic data of each config's shape and distribution, generated in HBM with
seeded torch generators; parameters per SURVEY.md §8(d) / Appendix C):

  c3  dense m=2000, n=4e6 (64 GB), w=8000, s=4, sigma=0.5
  c4  sparse m=1e4, n=2e7, 5 distinct rows/column (1e8 nnz, CSC), w=4e4, s=4, sigma=0.5
  c5  A = diag(r) G, r log-uniform [1e-3, 1e3], m=1000, n=2e6, Gaussian w=4000,
      sigma=0.3, repaired start (x0 log-uniform [1e-4, 1e4], s0 = U(0.5, 1.5) / x0)

Feasible start (x0, y0, s0) with b = A x0, c = A'y0 + s0, gamma_run =
max(gamma, 1 - 0.999 theta0), stop mu < 1e-8 max(1, mu0). One JSON line per
config.   python tools/solve_configs.py [c3] [c4] [c5]
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2209_08722_b200 import ipm_core as IC  # noqa: E402
from paper_2209_08722_b200 import kernels as K  # noqa: E402
from paper_2209_08722_b200.lp_model import DeviceLP  # noqa: E402
from paper_2209_08722_b200.runtime import F64, lda_for  # noqa: E402

DEV = torch.device("cuda")


def dense_cols(m, n, g, row_scale=None):
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=DEV)
    cols[:, :m].normal_(generator=g)
    if row_scale is not None:
        cols[:, :m] *= row_scale
    return K.DeviceMatrix(cols, m)


def sparse_cols(m, n, k, g):
    rows = torch.randint(0, m, (n, k), device=DEV, generator=g, dtype=torch.int64)
    for _ in range(64):  # redraw duplicates within a column until all rows are distinct
        rows, _ = torch.sort(rows, dim=1)
        dup = torch.zeros_like(rows, dtype=torch.bool)
        dup[:, 1:] = rows[:, 1:] == rows[:, :-1]
        nd = int(dup.sum().item())
        if nd == 0:
            break
        rows[dup] = torch.randint(0, m, (nd,), device=DEV, generator=g, dtype=torch.int64)
    vals = torch.randn((n, k), dtype=F64, device=DEV, generator=g)
    colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device=DEV)
    return K.SparseDeviceMatrix(colptr, rows.to(torch.int32).reshape(-1).contiguous(),
                                vals.reshape(-1), m)


def build(name):
    g = torch.Generator(device=DEV)
    g.manual_seed({"c3": 3, "c4": 4, "c5": 5}[name])
    if name == "c3":
        m, n = 2000, 4_000_000
        A = dense_cols(m, n, g)
        kw = dict(w=8000, s=4, sigma=0.5)
    elif name == "c4":
        m, n = 10_000, 20_000_000
        A = sparse_cols(m, n, 5, g)
        kw = dict(w=40_000, s=4, sigma=0.5)
    else:
        m, n = 1000, 2_000_000
        r = torch.exp(torch.empty(m, dtype=F64, device=DEV).uniform_(-6.907755, 6.907755,
                                                                      generator=g))
        A = dense_cols(m, n, g, row_scale=r)
        kw = dict(w=4000, sketch="gaussian", sigma=0.3)
    y0 = torch.randn(m, dtype=F64, device=DEV, generator=g)
    if name == "c5":
        x0 = torch.exp(torch.empty(n, dtype=F64, device=DEV).uniform_(-9.21034, 9.21034,
                                                                      generator=g))
        s0 = (torch.rand(n, dtype=F64, device=DEV, generator=g) + 0.5) / x0
    else:
        x0 = torch.rand(n, dtype=F64, device=DEV, generator=g) + 0.5
        s0 = torch.rand(n, dtype=F64, device=DEV, generator=g) + 0.5
    b = torch.empty(m, dtype=F64, device=DEV)
    K.gemv(A, x0, b)
    c = torch.empty(n, dtype=F64, device=DEV)
    K.gemv_t(A, y0, c, add=s0)
    lp = DeviceLP.from_device(A, b, c, n, name=name)
    return lp, x0, y0, s0, kw


def main(names):
    for name in names:
        lp, x0, y0, s0, kw = build(name)
        start = IC.make_iterate(lp, x0, y0, s0)
        gamma = max(0.1, 1.0 - 0.999 * start.min_xs / start.mu)
        prm = IC.IpmParams(mode="feasible", gamma=gamma, tol_outer=1e-8, seed=0, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = {"config": name, "m": lp.m, "n": lp.n, "sparse": lp.sparse, **kw,
               "gamma_run": round(gamma, 6)}
        try:
            rep = IC.solve(lp, start, prm)
            torch.cuda.synchronize()
            secs = time.perf_counter() - t0
            out.update(seconds=round(secs, 2), outer=rep.outer, sum_inner=rep.sum_inner,
                       max_inner=rep.max_inner, converged=rep.converged,
                       mu_final=rep.mu_final, objective=rep.objective,
                       ms_per_outer=round(secs * 1e3 / max(rep.outer, 1), 1))
        except Exception as e:  # report, do not hide
            out["error"] = f"{type(e).__name__}: {e}"[:300]
            out["seconds"] = round(time.perf_counter() - t0, 2)
        print(json.dumps(out), flush=True)
        del lp, x0, y0, s0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main([a for a in sys.argv[1:] if a in ("c3", "c4", "c5")] or ["c3", "c4", "c5"])
