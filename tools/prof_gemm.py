"""Event-timed DMMA GEMM shapes used by the factor (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
ws, cap = workspace(1 << 28)
def ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps * 1e3
for (M, N, K, lower) in [(960, 960, 64, 1), (960, 64, 64, 0), (512, 512, 64, 1), (64, 64, 64, 0),
                         (1000, 1000, 4000, 1), (4000, 1000, 1024, 0), (1024, 1024, 1024, 1)]:
    A = torch.randn((max(M, K), max(M, K)), dtype=torch.float64, device="cuda")
    B = torch.randn((max(N, K), max(N, K)), dtype=torch.float64, device="cuda")
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    us = ev(lambda: _lib.call("skb_gemm", 0, 1, M, N, K, 1.0, A, A.shape[1], B, B.shape[1], 0.0, C, N,
                              lower, 1, 0, 0, 0, ws, cap, stream_ptr()))
    tf = 2.0 * M * N * K / (2 if lower else 1) / (us * 1e-6) / 1e12
    tb = ev(lambda: torch.mm(A[:M, :K], B[:N, :K].t()))
    print(f"M={M} N={N} K={K} lower={lower}: {us:8.1f} us {tf:6.2f} TF/s   torch {tb:8.1f} us", flush=True)
C = torch.zeros((64, 64), dtype=torch.float64, device="cuda")
print("tiny fill kernel us", ev(lambda: C.zero_()))
x = torch.zeros(1000, dtype=torch.float64, device="cuda")
print("tiny add kernel us", ev(lambda: x.add_(1.0)))
A = torch.randn((64, 64), dtype=torch.float32, device="cuda")
print("fp32 64^3 mm us", ev(lambda: torch.mm(A, A)))
A = torch.randn((64, 64), dtype=torch.float64, device="cuda")
print("fp64 64^3 mm us", ev(lambda: torch.mm(A, A)))
