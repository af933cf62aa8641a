"""GPU busy vs wall for a few c2 outer steps via torch.profiler (CUPTI kernel
records; development aid)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.errors import MaxIterations
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for

m, n = 1000, 1_000_000
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(1000)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev)
cols[:, :m].normal_(generator=gen)
A = K.DeviceMatrix(cols, m)
x0 = torch.rand(n, dtype=F64, device=dev, generator=gen) + 0.5
s0 = torch.rand(n, dtype=F64, device=dev, generator=gen) + 0.5
g0 = torch.Generator(device=dev); g0.manual_seed(7)
y0 = torch.randn(m, dtype=F64, device=dev, generator=g0)
b = torch.empty(m, dtype=F64, device=dev); K.gemv(A, x0, b)
c = torch.empty(n, dtype=F64, device=dev); K.gemv_t(A, y0, c, add=s0)
lp = DeviceLP.from_device(A, b, c, n, name="c2")
start = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1.0 - 0.999 * start.min_xs / start.mu)
S = int(os.environ.get("PROF_S", 4))


def run(k):
    prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=4000, s=S, tol_outer=1e-8,
                       seed=0, max_outer=k)
    try:
        IC.solve(lp, start, prm)
    except MaxIterations:
        pass
    torch.cuda.synchronize()


run(2)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    run(4)
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in evs) / 1e3  # ms (kernel + memcpy/memset)
print(f"wall {wall * 1e3:.1f} ms for 4 outer; GPU busy {busy:.1f} ms ({busy / (wall * 1e3):.0%}); "
      f"{len(evs)} device ops")
agg = {}
for e in evs:
    k = e.name[:60]
    t, c_ = agg.get(k, (0.0, 0))
    agg[k] = (t + e.device_time / 1e3, c_ + 1)
for k, (t, c_) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{t:9.3f} ms  n={c_:5d}  {k}")
norm = sorted(e.device_time for e in evs if "OpNormal" in e.name)
print("OpNormal durations (us): min %.1f  p10 %.1f  p50 %.1f  p90 %.1f  max %.1f" % (
    norm[0], norm[len(norm) // 10], norm[len(norm) // 2], norm[9 * len(norm) // 10], norm[-1]))
print("gated-looking (<100 us):", sum(1 for t in norm if t < 100), "sum us", sum(t for t in norm if t < 100))
# idle gaps between consecutive device ops (> 15 us), attributed to the op after the gap
ops = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
gaps = collections.Counter() if False else {}
import collections as _c
gsum = _c.Counter(); gcnt = _c.Counter()
allgap = 0.0
for (s0, e0, n0), (s1, e1, n1) in zip(ops, ops[1:]):
    gap = s1 - e0
    allgap += max(gap, 0)
    if gap > 15:
        key = n0[:40] + " -> " + n1[:40]
        gsum[key] += gap; gcnt[key] += 1
tot = sum(gsum.values())
print(f"idle gaps > 15 us: {tot / 1e3:.2f} ms total over 4 outer; all gaps {allgap / 1e3:.2f} ms")
for k, v in gsum.most_common(15):
    print(f"{v / 1e3:8.3f} ms  n={gcnt[k]:4d}  {k}")
