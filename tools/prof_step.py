"""Time c2 outer steps (s configurable) and break down where the time goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_08722_b200 import ipm_core as IC, kernels as K
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for
m, n = 1000, int(os.environ.get("PROF_N", 1_000_000))
s_nnz = int(os.environ.get("PROF_S", 4)); steps = int(os.environ.get("PROF_STEPS", 6))
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(1000)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev); cols[:, :m].normal_(generator=gen)
A = K.DeviceMatrix(cols, m)
x0 = torch.rand(n, dtype=F64, device=dev, generator=gen) + 0.5
s0 = torch.rand(n, dtype=F64, device=dev, generator=gen) + 0.5
y0 = torch.randn(m, dtype=F64, device=dev, generator=gen)
b = torch.empty(m, dtype=F64, device=dev); K.gemv(A, x0, b)
c = torch.empty(n, dtype=F64, device=dev); K.gemv_t(A, y0, c, add=s0)
lp = DeviceLP.from_device(A, b, c, n)
it = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1 - 0.999 * it.min_xs / it.mu)
prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=4000, s=s_nnz, tol_outer=1e-8)
rng = np.random.Generator(np.random.Philox(0))
for k in range(steps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    it, rec = IC.ipm_step(lp, it, prm, rng, None, None)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"step {k}: {1e3*(t1-t0):.2f} ms  inner {rec.inner_iterations} total {rec.inner_iterations_total} vret {rec.v_retries}", flush=True)
