"""c2 solve, a few outer steps, wall time per step (development aid; run under
ncu --metrics gpu__time_duration.sum for the per-kernel split)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.errors import MaxIterations
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for

m, n = 1000, int(os.environ.get("PROF_N", 1_000_000))
steps = int(os.environ.get("PROF_STEPS", 4))
s_nnz = int(os.environ.get("PROF_S", 4))
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
times = []
def on_step(rec):
    torch.cuda.synchronize(); times.append(time.perf_counter())
def run(k):
    prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=4000, s=s_nnz, tol_outer=1e-8,
                       seed=0, max_outer=k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        rep = IC.solve(lp, start, prm)
    except MaxIterations as e:
        rep = e.report
    torch.cuda.synchronize()
    return time.perf_counter() - t0, rep

run(1)  # warm-up (workspaces, first launches)
t_a, rep_a = run(2)
t_b, rep_b = run(2 + steps)
print(f"{steps} outer steps (after 2): {(t_b - t_a) * 1e3 / steps:.2f} ms/outer; "
      f"inner {[r.inner_iterations for r in rep_b.steps]}")
