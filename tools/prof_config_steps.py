"""GPU busy vs wall for a few outer steps of c3 / c4 / c5 (torch.profiler CUPTI
kernel records) with the top kernels; development aid.
    python tools/prof_config_steps.py c4"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import solve_configs as SC
from paper_2209_08722_b200 import ipm_core as IC

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
lp, x0, y0, s0, kw = SC.build(name)
it = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1.0 - 0.999 * it.min_xs / it.mu)
prm = IC.IpmParams(mode="feasible", gamma=gamma, tol_outer=1e-8, seed=0, **kw)
rng = np.random.Generator(np.random.Philox(0))
for _ in range(2):
    it, rec = IC.ipm_step(lp, it, prm, rng, None, None)
torch.cuda.synchronize()
K = 3
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    for _ in range(K):
        it, rec = IC.ipm_step(lp, it, prm, rng, None, None)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in evs) / 1e3
print(f"{name}: {1e3 * wall / K:.1f} ms wall per outer step, GPU busy {busy / K:.1f} ms "
      f"({busy / (wall * 1e3):.0%})")
agg = {}
for e in evs:
    k = e.name[:70]
    t, c_ = agg.get(k, (0.0, 0))
    agg[k] = (t + e.device_time / 1e3, c_ + 1)
for k, (t, c_) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:18]:
    print(f"{t / K:9.3f} ms/step  n={c_ / K:6.1f}  {k}")
