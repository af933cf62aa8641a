"""Kernel-time breakdown and idle gaps of K outer steps of a full-size config
(c3 / c4 / c5 from tools/solve_configs.py) via torch.profiler (development aid).
    python tools/prof_config_timeline.py c4 [K]"""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import solve_configs as SC
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200.errors import MaxIterations

name = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lp, x0, y0, s0, kw = SC.build(name)
start = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1.0 - 0.999 * start.min_xs / start.mu)


def run(kk):
    prm = IC.IpmParams(mode="feasible", gamma=gamma, tol_outer=1e-8, seed=0, max_outer=kk, **kw)
    try:
        IC.solve(lp, start, prm)
    except MaxIterations:
        pass
    torch.cuda.synchronize()


run(1)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    run(k)
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in evs) / 1e3
print(f"{name}: wall {wall * 1e3:.1f} ms for {k} outer (incl. solve setup); GPU busy {busy:.1f} ms")
agg = collections.defaultdict(lambda: [0.0, 0])
for e in evs:
    a = agg[e.name[:70]]
    a[0] += e.device_time / 1e3
    a[1] += 1
for kname, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:22]:
    print(f"{t:9.2f} ms  n={c:5d}  {kname}")
ops = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
gsum = collections.Counter(); gcnt = collections.Counter()
for (s0_, e0, n0), (s1, e1, n1) in zip(ops, ops[1:]):
    if s1 - e0 > 20:
        key = n0[:35] + " -> " + n1[:35]
        gsum[key] += s1 - e0; gcnt[key] += 1
print(f"idle gaps > 20 us: {sum(gsum.values()) / 1e3:.1f} ms")
for kname, v in gsum.most_common(8):
    print(f"{v / 1e3:8.2f} ms  n={gcnt[kname]:4d}  {kname}")
