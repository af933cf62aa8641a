"""Host-side gap accounting for c2 outer steps: wall time between consecutive
host synchronisations (to_host readbacks and the C-level readbacks) and where
they happen. Development aid."""
import collections, os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200 import runtime as RT
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for

m, n = 1000, int(os.environ.get("PROF_N", 1_000_000))
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(1000)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev)
cols[:, :m].normal_(generator=gen)
A = K.DeviceMatrix(cols, m)
x0 = torch.rand(n, dtype=F64, device=dev, generator=gen) + 0.5
s0 = torch.rand(n, dtype=F64, device=dev, generator=gen) + 0.5
y0 = torch.randn(m, dtype=F64, device=dev, generator=gen)
b = torch.empty(m, dtype=F64, device=dev); K.gemv(A, x0, b)
c = torch.empty(n, dtype=F64, device=dev); K.gemv_t(A, y0, c, add=s0)
lp = DeviceLP.from_device(A, b, c, n, name="c2")
it = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1.0 - 0.999 * it.min_xs / it.mu)
prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=4000, s=4, tol_outer=1e-8, seed=0)
rng = np.random.Generator(np.random.Philox(0))

events = []
orig_to_host = RT.to_host
def to_host(t):
    t0 = time.perf_counter()
    out = orig_to_host(t)
    t1 = time.perf_counter()
    st = traceback.extract_stack(limit=4)[-3]
    events.append(("to_host", f"{os.path.basename(st.filename)}:{st.lineno}", t0, t1))
    return out
orig_call = _lib.call
def call(name, *a):
    t0 = time.perf_counter()
    r = orig_call(name, *a)
    t1 = time.perf_counter()
    if t1 - t0 > 200e-6:
        events.append(("call", name, t0, t1))
    return r
for mod in list(sys.modules.values()):
    if mod and getattr(mod, "__name__", "").startswith("paper_2209_08722_b200"):
        if getattr(mod, "to_host", None) is orig_to_host:
            mod.to_host = to_host
_lib.call = call

for k in range(3):
    it, rec = IC.ipm_step(lp, it, prm, rng, None, None)
torch.cuda.synchronize()
events.clear()
T0 = time.perf_counter()
for k in range(2):
    it, rec = IC.ipm_step(lp, it, prm, rng, None, None)
torch.cuda.synchronize()
T1 = time.perf_counter()
print(f"2 outer steps: {1e3 * (T1 - T0):.1f} ms wall; {len(events)} blocking events")
agg = collections.defaultdict(lambda: [0, 0.0])
for kind, where, t0, t1 in events:
    agg[f"{kind} {where}"][0] += 1
    agg[f"{kind} {where}"][1] += t1 - t0
for k, (cnt, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{1e3 * t:8.2f} ms  n={cnt:3d}  {k}")
