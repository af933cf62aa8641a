"""One c5 Gaussian-sketch product X = (A D W)' (m=1000, n=2e6, w=4000) between
cudaProfilerStart/Stop, for an ncu launch list (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import F64, lda_for, stream_ptr, workspace
m, n, w = 1000, int(os.environ.get("PROF_N", 2_000_000)), 4000
g = torch.Generator(device="cuda"); g.manual_seed(5)
A = torch.randn((n, lda_for(m)), dtype=F64, device="cuda", generator=g)
d = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.5
W = torch.randn((n, w), dtype=F64, device="cuda", generator=g)
X = torch.empty((w, lda_for(m)), dtype=F64, device="cuda")
ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(m, w)) + (8 << 30))
def run():
    _lib.call("skb_gaussian_apply", A, m, n, lda_for(m), d, W, w, X, lda_for(m), ws, cap, stream_ptr())
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); e1.synchronize()
print(f"c5 product: {e0.elapsed_time(e1):.2f} ms")
torch.cuda.profiler.start(); run(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
