"""GPU busy vs wall and the largest idle gaps of a CholeskyQR2 factor build at
(PROF_M, PROF_W) via torch.profiler (CUPTI; development aid)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2209_08722_b200.kernels import DeviceMatrix
from paper_2209_08722_b200 import preconditioning as PC
m, w = int(os.environ.get("PROF_M", 10000)), int(os.environ.get("PROF_W", 40000))
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = DeviceMatrix(torch.randn((w, m + (m & 1)), dtype=torch.float64, device="cuda", generator=g), m)
PC.build_preconditioner(X); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    PC.build_preconditioner(X); torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in evs) / 1e3
print(f"wall {wall * 1e3:.1f} ms; GPU busy {busy:.1f} ms ({busy / (wall * 1e3):.0%}); {len(evs)} device ops")
ops = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
gsum = collections.Counter(); gcnt = collections.Counter()
for (s0, e0, n0), (s1, e1, n1) in zip(ops, ops[1:]):
    gap = s1 - e0
    if gap > 10:
        key = n0[:45] + " -> " + n1[:45]
        gsum[key] += gap; gcnt[key] += 1
print(f"idle gaps > 10 us: {sum(gsum.values()) / 1e3:.2f} ms")
for k, v in gsum.most_common(20):
    print(f"{v / 1e3:8.3f} ms  n={gcnt[k]:4d}  {k}")
