"""Probe: int8 x int8 -> int32 tensor-core GEMM throughput (cuBLASLt via torch._int_mm)."""
import torch
for (M, N, K) in [(4096, 4096, 4096), (8192, 8192, 8192), (10000 // 16 * 16, 10000 // 16 * 16, 40000), (1024, 4096, 65536)]:
    a = torch.randint(-128, 127, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (N, K), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        c = torch._int_mm(a, b)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(M, N, K, "ms %.3f  TOPS %.1f" % (ms, 2 * M * N * K / ms / 1e9))
x = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): y = x @ x
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); y = x @ x; e1.record(); e1.synchronize()
print("cublas dgemm 8192^3 TF %.1f" % (2 * 8192**3 / e0.elapsed_time(e1) / 1e9))
