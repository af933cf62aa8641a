"""c2 Gram G = X'X (X = ADW', 4000 x 1000): our lower-tile DMMA SYRK (skb_gemm) vs
cuBLAS DGEMM through torch.matmul (full product), CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import stream_ptr, workspace
for (w, m) in ((4000, 1000), (8000, 2000)):
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    X = torch.randn((w, m), dtype=torch.float64, device="cuda", generator=g)
    G = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(m, w)))
    os.environ["SKB_GEMM_EMU"] = "0"
    def ours():
        _lib.call("skb_gemm", 1, 0, m, m, w, 1.0, X, m, X, m, 0.0, G, m, 1, 1, 0, 0, 0, ws, cap, stream_ptr())
    def cub():
        torch.matmul(X.t(), X)
    for name, fn, fl in (("ours lower-tile SYRK (DMMA)", ours, m * (m + 1) * w), ("cuBLAS DGEMM full", cub, 2 * m * m * w)):
        for _ in range(3): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(20): fn()
        b.record(); b.synchronize()
        ms = a.elapsed_time(b) / 20
        print(f"{m}x{m}x{w} {name}: {ms:.4f} ms, {fl / ms / 1e9:.1f} TF/s on its own flops, "
              f"{m * (m + 1) * w / ms / 1e9:.1f} TF/s on the Gram's lower flops")
