"""CUDA-event time of each fused A-pass at c2 (or PROF_M / PROF_N) size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.runtime import F64, lda_for
m, n = int(os.environ.get("PROF_M", 1000)), int(os.environ.get("PROF_N", 1_000_000))
dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(0)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev); cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
vec = lambda k: torch.rand(k, dtype=F64, device=dev, generator=g) + 0.5  # noqa: E731
x, s, v, c, d2, dx, ds = (vec(n) for _ in range(7))
z, y, b = vec(m), vec(m), vec(m)
outm = torch.empty(m, dtype=F64, device=dev)
o1, o2, o3 = (torch.empty(n, dtype=F64, device=dev) for _ in range(3))


def ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    e.record(); e.synchronize()
    return a.elapsed_time(e) / reps


for name, fn in [
    ("normal", lambda: K.normal_apply(A, d2, z, outm)),
    ("directions", lambda: K.directions(A, y, x, s, v, 0.3, o1, o2, outm, atdy=o3)),
    ("iterate", lambda: K.iterate(A, x, s, y, b, c, outm, o1, dx=dx, ds=ds, alpha=0.5, x_out=o2,
                                  s_out=o3)),
    ("rhs", lambda: K.rhs(A, x, s, 0.3, outm)),
    ("gemv_ratio", lambda: K.gemv_ratio(A, v, s, outm)),
]:
    print(f"{name:12s} {ev(fn):.4f} ms", flush=True)
