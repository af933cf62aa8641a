"""One large DMMA GEMM (PROF_SHAPE=M,N,K,ta,tb) for ncu (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
M, N, K, ta, tb = map(int, os.environ.get("PROF_SHAPE", "4096,4096,4096,0,0").split(","))
Am = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
Bm = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda")
C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
ws, cap = workspace(1 << 28)
for _ in range(2):
    _lib.call("skb_gemm", ta, tb, M, N, K, 1.0, Am, Am.shape[1], Bm, Bm.shape[1], 0.0, C, N, 0, 1,
              0, 0, 0, ws, cap, stream_ptr())
torch.cuda.synchronize()
print("ok")
