"""Count host<->device synchronisations in one c2-like outer step (torch sync
debug mode; small n so it runs fast). Development aid."""
import os, sys, warnings, collections, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import ipm_core as IC
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.errors import MaxIterations
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for

m, n = 1000, 100_000
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
lp = DeviceLP.from_device(A, b, c, n, name="c2s")
start = IC.make_iterate(lp, x0, y0, s0)
gamma = max(0.1, 1.0 - 0.999 * start.min_xs / start.mu)
rng = __import__("numpy").random.Generator(__import__("numpy").random.Philox(0))
prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=4000, s=4, tol_outer=1e-8, seed=0)
IC.ipm_step(lp, start, prm, rng, start.residual_norm, start.mu)   # warm
torch.cuda.synchronize()
sites = collections.Counter()
def hook(message, category, filename, lineno, file=None, line=None):
    st = traceback.extract_stack()
    for fr in reversed(st):
        if "paper_2209_08722_b200" in fr.filename:
            sites[f"{os.path.basename(fr.filename)}:{fr.lineno} {fr.line}"] += 1
            break
warnings.showwarning = hook
warnings.simplefilter("always")
torch.cuda.set_sync_debug_mode(1)
IC.ipm_step(lp, start, prm, rng, start.residual_norm, start.mu)
torch.cuda.set_sync_debug_mode(0)
print("torch-visible syncs:", sum(sites.values()))
for k, v in sites.most_common():
    print(f"{v:4d}  {k}")
