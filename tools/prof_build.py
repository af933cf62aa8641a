"""c2 sketch + factor build for launch-list profiling (m=1000, n=1e6, w=4000)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K, sketching as S, preconditioning as PC
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import lda_for

m, n, w = 1000, int(os.environ.get("PROF_N", 1_000_000)), 4000
s = int(os.environ.get("PROF_S", 1))
g = torch.Generator(device="cuda"); g.manual_seed(0)
cols = torch.zeros((n, lda_for(m)), dtype=torch.float64, device="cuda")
cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
b = torch.zeros(m, dtype=torch.float64, device="cuda")
c = torch.ones(n, dtype=torch.float64, device="cuda")
lp = DeviceLP.from_device(A, b, c, n)
d = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
for rep in range(int(os.environ.get("PROF_REPS", 3))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    W = S.build_sparse_embedding(n, w, s, 100 + rep)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    X = S.apply_sketch(lp, d, W, check_positive=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    f = PC.build_preconditioner(X)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"s={s} hash {1e3*(t1-t0):.3f} ms  adw {1e3*(t2-t1):.3f} ms  factor {1e3*(t3-t2):.3f} ms", flush=True)
