"""Minimal c2 workload for ncu: one fused A D^2 A' z pass repeated (m=1000, n=1e6)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.runtime import lda_for

m, n = int(os.environ.get("PROF_M", 1000)), int(os.environ.get("PROF_N", 1_000_000))
g = torch.Generator(device="cuda"); g.manual_seed(0)
cols = torch.zeros((n, lda_for(m)), dtype=torch.float64, device="cuda")
cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
d2 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
z = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
u = torch.empty(m, dtype=torch.float64, device="cuda")
t = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("PROF_REPS", 5))):
    K.normal_apply(A, d2, z, u)
    K.gemv_t(A, z, t)
    K.gemv(A, d2, u)
torch.cuda.synchronize()
print("ok")
