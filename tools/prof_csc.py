"""c4 CSC normal pass: planned (cscp_kernel) vs atomic (csc_kernel), CUDA-event times."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2209_08722_b200 import kernels as K  # noqa: E402
from paper_2209_08722_b200.runtime import F64  # noqa: E402

m, n, k = 10_000, 20_000_000, 5
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = torch.Generator(device="cuda")
g.manual_seed(4)
base = torch.randint(0, m // k, (n, k), device="cuda", generator=g, dtype=torch.int32)
rows = (base + torch.arange(k, device="cuda", dtype=torch.int32) * (m // k)).reshape(-1).contiguous()
vals = torch.randn(n * k, dtype=F64, device="cuda", generator=g)
colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device="cuda")
A = K.SparseDeviceMatrix(colptr, rows, vals, m)
B = K.SparseDeviceMatrix(colptr, rows, vals, m)
B._plan = (None, 0)
Cm = K.SparseDeviceMatrix(colptr, rows, vals, m)
Cm._plan = (None, 0)
Cm._ell = None
d2 = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.5
z = torch.randn(m, dtype=F64, device="cuda", generator=g)
u = torch.empty(m, dtype=F64, device="cuda")
t0 = time.perf_counter()
A.plan(force=True)
torch.cuda.synchronize()
print(f"plan build {1e3 * (time.perf_counter() - t0):.1f} ms, chunks {A.plan()[1]}")
byt = 12 * n * k + 16 * n + 8 + 16 * m
for name, M in (("planned", A), ("atomic+ell", B), ("atomic", Cm)):
    for _ in range(3):
        K.normal_apply(M, d2, z, u)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        K.normal_apply(M, d2, z, u)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: {ms:.4f} ms  {byt / ms / 1e6:.1f} GB/s")
