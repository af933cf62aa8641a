"""Event-timed dense normal apply at m = 2000 (c3 per-GPU shape, n = 2e6)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.runtime import F64, lda_for
m, n = int(os.environ.get("PROF_M", 2000)), int(os.environ.get("PROF_N", 2_000_000))
g = torch.Generator(device="cuda"); g.manual_seed(0)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device="cuda"); cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
d2 = torch.rand(n, dtype=F64, device="cuda", generator=g)
z = torch.randn(m, dtype=F64, device="cuda", generator=g); u = torch.empty(m, dtype=F64, device="cuda")
for _ in range(3): K.normal_apply(A, d2, z, u)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): K.normal_apply(A, d2, z, u)
b.record(); b.synchronize()
ms = a.elapsed_time(b) / 10
print(f"m={m} n={n}: {ms:.3f} ms  {(8.0*m*n + 16*n + 16*m)/ms/1e6:.0f} GB/s  env CPS={os.environ.get('SKB_COOP_CPS')} KB={os.environ.get('SKB_COOP_STAGE_KB')}")
