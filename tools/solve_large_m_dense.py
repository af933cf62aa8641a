"""A dense LP past the staged kernels' shared-memory ceilings (m = 15,000): a few outer
steps end to end on the device (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.errors import MaxIterations
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for
m = int(os.environ.get("PM", 15000)); n = 8 * m
dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(1)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev); cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
x0 = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.5
s0 = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.5
y0 = torch.randn(m, dtype=F64, device=dev, generator=g)
b = torch.empty(m, dtype=F64, device=dev); K.gemv(A, x0, b)
c = torch.empty(n, dtype=F64, device=dev); K.gemv_t(A, y0, c, add=s0)
lp = DeviceLP.from_device(A, b, c, n, name="large_m_dense")
it = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1.0 - 0.999 * it.min_xs / it.mu)
prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=2 * m, s=4, tol_outer=1e-8, seed=0,
                   max_outer=int(os.environ.get("PK", 3)))
t0 = time.perf_counter()
try:
    steps = IC.solve(lp, it, prm).steps
except MaxIterations as e:
    steps = e.report.steps
print(f"dense m={m} n={n}: {len(steps)} outer steps in {time.perf_counter() - t0:.1f} s, mu "
      + ", ".join(f"{r.mu_after:.3e}" for r in steps) + f"; inner {[r.inner_iterations for r in steps]}",
      flush=True)
