"""One emulated GEMM (shape from argv: ta tb M N K lower) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
ta, tb, M, N, K, low = (int(v) for v in sys.argv[1:7])
g = torch.Generator(device="cuda"); g.manual_seed(0)
A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
B = A if (ta != tb and M == N and "share" in sys.argv) else torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
ws, cap = workspace(int(_lib.lib().skb_gemm_ozaki_workspace_bytes(M, N, min(K, 65536))) + (64 << 20))
for _ in range(2):
    _lib.call("skb_gemm_ozaki", ta, tb, M, N, K, 1.0, A, A.shape[1], B, B.shape[1], 0.0, C, N, low,
              ws, cap, stream_ptr())
torch.cuda.synchronize()
