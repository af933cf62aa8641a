"""Host-side call sequence with time deltas for one c2 outer step: large deltas
between consecutive library calls are host work while the GPU may idle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.argv = [sys.argv[0]]
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_solve_timeline.py")).read()
exec(src.split("run(2)")[0])
from paper_2209_08722_b200 import _lib
log = []
orig = _lib.call
def wrapped(name, *a):
    t0 = time.perf_counter()
    r = orig(name, *a)
    log.append((t0, time.perf_counter(), name))
    return r
_lib.call = wrapped
orig_cpu = torch.Tensor.cpu
def cpu(self, *a, **k):
    t0 = time.perf_counter()
    r = orig_cpu(self, *a, **k)
    log.append((t0, time.perf_counter(), "cpu()"))
    return r
torch.Tensor.cpu = cpu
run(2)
log.clear()
run(3)
prev = log[0][1]
rows = []
for t0, t1, name in log:
    rows.append((t0 - prev, t1 - t0, name))
    prev = t1
big = sorted(rows, key=lambda r: -r[0])[:25]
print("largest host gaps before a call (us), call duration (us), call:")
for g, d, n in big:
    print(f"{g * 1e6:9.1f} {d * 1e6:9.1f}  {n}")
print("sum of gaps (ms):", sum(r[0] for r in rows) * 1e3, "calls", len(rows))
# the ordered sequence of one step (largest gaps flagged)
print("--- sequence (gap_us, dur_us, call) for the first ~70 calls of the 2nd step ---")
marks = [i for i, (_, _, nm) in enumerate(log) if nm == "skb_step_prep"]
if len(marks) >= 2:
    i0, i1 = marks[1], marks[2] if len(marks) > 2 else len(log)
    prev = log[i0 - 1][1]
    for t0, t1, nm in log[i0 - 3:i1]:
        print(f"{(t0 - prev) * 1e6:9.1f} {(t1 - t0) * 1e6:9.1f}  {nm}")
        prev = t1
