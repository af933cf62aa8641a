"""A sparse LP past the shared-memory CSC kernels' ceiling (m = 16,000): a few outer
steps end to end on the device (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200.errors import MaxIterations
from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
from paper_2209_08722_b200.problems import sparse_wide_lp
m = int(os.environ.get("PM", 16000))
lpd = sparse_wide_lp(m, 6 * m, 5, 3)
dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c))
kw = dict(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=2 * m, s=4, tol_outer=1e-8,
          seed=1, max_outer=int(os.environ.get("PK", 4)))
t0 = time.perf_counter()
try:
    rep = IC.solve(dlp, IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0), IC.IpmParams(**kw))
    steps = rep.steps
except MaxIterations as e:
    steps = e.report.steps
print(f"m={m}: {len(steps)} outer steps in {time.perf_counter() - t0:.1f} s, mu "
      + ", ".join(f"{r.mu_after:.3e}" for r in steps)
      + f"; inner {[r.inner_iterations for r in steps]}", flush=True)
