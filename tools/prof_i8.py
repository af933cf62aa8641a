"""tcgen05 INT8 batched GEMM (skb_i8gemm_batched) throughput, and the whole
emulated FP64 GEMM (skb_gemm_ozaki) with the INT8 products on this kernel vs
cuBLASLt (SKB_OZ_CUBLASLT=1). CUDA events, after warm-up."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2209_08722_b200 import _lib  # noqa: E402
from paper_2209_08722_b200.runtime import stream_ptr, workspace  # noqa: E402


def ev(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for (n, R, Kp) in [(16, 4096, 8192), (16, 8192, 16384), (16, 1280, 40960)]:
    A = torch.randint(-128, 128, (n, R, Kp), dtype=torch.int8, device="cuda")
    C = torch.empty((n, R, R), dtype=torch.int32, device="cuda")
    f = lambda: _lib.call("skb_i8gemm_batched", A, R, R * Kp, A, R, R * Kp, Kp, C, R, R * R, R,  # noqa
                          R, 0, 0, 0, Kp, n, 0, 0, stream_ptr())
    ms = ev(f, 5)
    print(f"i8gemm n={n} {R}x{R}x{Kp}: {ms:.3f} ms  {2.0 * n * R * R * Kp / ms / 1e9:.1f} TOPS")
    del A, C
    torch.cuda.empty_cache()

for (M, N, K, lower) in [(10000, 10000, 40000, 1), (4000, 10000, 10000, 0), (1000, 4000, 2000000, 0)]:
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = A if (M == N and lower) else torch.randn(N, K, dtype=torch.float64, device="cuda",
                                                    generator=g)
    C = torch.zeros(M, N, dtype=torch.float64, device="cuda")
    need = int(_lib.lib().skb_gemm_ozaki_workspace_bytes(M, N, K))
    ws, cap = workspace(need)
    for route in ("0", "1"):
        os.environ["SKB_OZ_CUBLASLT"] = route
        f = lambda: _lib.call("skb_gemm_ozaki", 0, 1, M, N, K, 1.0, A, K, B, K, 0.0, C, N,  # noqa
                              lower, ws, cap, stream_ptr())
        ms = ev(f, 2)
        fl = 2.0 * M * N * K * (0.5 if lower else 1.0)
        print(f"ozaki {M}x{N}x{K} lower={lower} {'cublasLt' if route == '1' else 'tcgen05 '}: "
              f"{ms:.2f} ms  {fl / ms / 1e9:.1f} TF/s fp64-equiv")
    del A, B, C
    torch.cuda.empty_cache()
