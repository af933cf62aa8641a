import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.runtime import F64
dev = torch.device("cuda")
m, n, k = 10_000, 20_000_000, 5
g = torch.Generator(device=dev); g.manual_seed(4)
rows = torch.randint(0, m, (n, k), device=dev, generator=g, dtype=torch.int32)
rows, _ = torch.sort(rows, dim=1)
vals = torch.randn((n, k), dtype=F64, device=dev, generator=g)
colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device=dev)
A = K.SparseDeviceMatrix(colptr, rows.reshape(-1).contiguous(), vals.reshape(-1), m)
x = torch.rand(n, dtype=F64, device=dev, generator=g)
y = torch.randn(m, dtype=F64, device=dev, generator=g)
u = torch.empty(m, dtype=F64, device=dev); t = torch.empty(n, dtype=F64, device=dev)
def ev(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps
print("normal (dot+axpy):", ev(lambda: K.normal_apply(A, x, y, u)))
print("gemv_t (dot only):", ev(lambda: K.gemv_t(A, y, t)))
print("gemv (axpy only): ", ev(lambda: K.gemv(A, x, u)))
