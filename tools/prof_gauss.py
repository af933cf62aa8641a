"""Event-timed K9 Gaussian sketch generation (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
n, w = int(os.environ.get("PROF_N", 50_000)), 4000
W = torch.empty((n, w), dtype=torch.float64, device="cuda")
extra = int(_lib.lib().skb_gaussian_value_bytes(n * w)) if os.environ.get("SKB_ZIG_STORE", "1") != "0" else 0
ws, cap = workspace(int(_lib.lib().skb_gaussian_workspace_bytes(n * w)) + extra)
def gen():
    _lib.call("skb_gaussian_sketch", 123, 456, 0, n * w, w, W, ws, cap, stream_ptr())
gen(); torch.cuda.synchronize()
reps = int(os.environ.get("PROF_REPS", 5))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps): gen()
b.record(); b.synchronize()
ms = a.elapsed_time(b) / reps
print(f"n={n} w={w}: {ms:.3f} ms  {n*w/ms/1e6:.3e} draws/s  {8*n*w/ms/1e6:.1f} GB/s written")
