"""Dump device solve records for a golden case (development diagnostic)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
from paper_2209_08722_b200.problems import wide_dense_lp

out = {}
lpd = wide_dense_lp(40, 3000, 5)
dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c))
st = IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0)
rep = IC.solve(dlp, st, IC.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=160,
                                      s=4, tol_outer=1e-7, seed=3))
out["small_feasible"] = rep.to_dict()
out["small_feasible"].pop("params")
lpd = wide_dense_lp(100, 10_000, 0)
dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c))
st = IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0)
rep = IC.solve(dlp, st, IC.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=400,
                                      s=1, tol_outer=1e-6, seed=0))
out["c1_s1"] = rep.to_dict()
out["c1_s1"].pop("params")
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/diag_trace.json", "w"))
print("done", out["small_feasible"]["outer"], out["c1_s1"]["outer"])
