"""Quick device timing of the streaming kernels (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.runtime import lda_for

def timeit(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters

for (m, n) in [(1000, 1_000_000), (100, 10_000_000), (2000, 500_000), (1000, 100_000)]:
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    cols = torch.randn((n, lda_for(m)), dtype=torch.float64, device="cuda", generator=g)
    A = K.DeviceMatrix(cols, m)
    d2 = torch.rand(n, dtype=torch.float64, device="cuda") + 0.5
    z = torch.randn(m, dtype=torch.float64, device="cuda")
    u = torch.empty(m, dtype=torch.float64, device="cuda")
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    byt = 8.0 * m * n + 8 * n + 16 * m
    ms = timeit(lambda: K.normal_apply(A, d2, z, u))
    print(f"normal m={m} n={n}: {ms:.3f} ms  {byt/ms/1e6:.1f} GB/s", flush=True)
    ms = timeit(lambda: K.gemv_t(A, z, t))
    print(f"gemv_t m={m} n={n}: {ms:.3f} ms  {(8.0*m*n+8*n)/ms/1e6:.1f} GB/s", flush=True)
    ms = timeit(lambda: K.gemv(A, d2, u))
    print(f"gemv   m={m} n={n}: {ms:.3f} ms  {(8.0*m*n+8*n)/ms/1e6:.1f} GB/s", flush=True)
    del cols, A
    torch.cuda.empty_cache()
