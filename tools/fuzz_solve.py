"""Randomized whole-solve parity sweep: device solve vs the pinned oracle (the
reference algorithm restated, oracle/ipm_oracle.py) on random wide LPs —
dense, sparse (CSC path), ill-conditioned, Gaussian sketch, other inner
solvers. Reports outer / inner counts, sketch seeds and the objective
(development aid; the GPU tests gate the fixed cases)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from oracle import ipm_oracle as O
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
from paper_2209_08722_b200.problems import ill_conditioned_lp, sparse_wide_lp, wide_dense_lp

rng = np.random.default_rng(int(os.environ.get("FUZZ_SEED", 3)))
rows = []
for case in range(int(os.environ.get("FUZZ_N", 12))):
    kind = ["dense", "sparse", "illcond", "gaussian", "chebyshev", "direct"][case % 6]
    m = int(rng.integers(12, 70))
    n = int(rng.integers(40 * m, 80 * m))
    seed = int(rng.integers(0, 1000))
    if kind == "sparse":
        lpd = sparse_wide_lp(m, n, 5, seed)
    elif kind == "illcond":
        lpd = ill_conditioned_lp(m, n, seed)
    else:
        lpd = wide_dense_lp(m, n, seed)
    kw = dict(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5 if kind != "illcond" else 0.3,
              w=4 * m, s=4, tol_outer=1e-6, seed=int(rng.integers(0, 100)))
    if kind == "gaussian":
        kw["sketch"] = "gaussian"
    if kind in ("chebyshev", "direct"):
        kw["solver"] = kind
        if kind == "chebyshev":
            kw["w"], kw["s"] = 30 * m, 12
    A = lpd.A if sp.issparse(lpd.A) else np.asarray(lpd.A)
    dlp = DeviceLP.from_host(LinearProgram(A, lpd.b, lpd.c))
    rep = IC.solve(dlp, IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0), IC.IpmParams(**kw))
    Ac = sp.csr_matrix(A)
    orp = O.solve(Ac, lpd.b, lpd.c, O.make_iterate(Ac, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0),
                  O.Params(**kw))
    ref = orp if isinstance(orp, dict) else orp.__dict__
    g_outer = ref["outer"] if "outer" in ref else len(ref["steps"])
    g_inner = [s["inner_iterations"] if isinstance(s, dict) else s.inner_iterations
               for s in ref["steps"]]
    g_obj = ref["objective"]
    d_inner = [r.inner_iterations for r in rep.steps]
    same_inner = d_inner == g_inner
    obj_rel = abs(rep.objective - g_obj) / max(abs(g_obj), 1e-300)
    ok = rep.outer == g_outer and obj_rel <= 1e-8
    rows.append(ok)
    print(f"case {case} {kind:9s} m={m} n={n}: outer {rep.outer}/{g_outer} inner-identical={same_inner} "
          f"obj rel {obj_rel:.1e} ok={ok}", flush=True)
print("OK", sum(rows), "of", len(rows))
