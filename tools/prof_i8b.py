"""One emulated FP64 Gram (10000 x 10000 x 40000, lower) per INT8 route, for a
launch list under ncu (route via argv: 0 = tcgen05 kernel, 1 = cuBLASLt)."""
import os
import sys

import torch

sys.path.insert(0, ".")
os.environ["SKB_OZ_CUBLASLT"] = sys.argv[1] if len(sys.argv) > 1 else "0"
from paper_2209_08722_b200 import _lib  # noqa: E402
from paper_2209_08722_b200.runtime import stream_ptr, workspace  # noqa: E402

M = N = 10000
K = 40000
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(M, N, dtype=torch.float64, device="cuda")
ws, cap = workspace(int(_lib.lib().skb_gemm_ozaki_workspace_bytes(M, N, K)))
for _ in range(2):
    _lib.call("skb_gemm_ozaki", 0, 1, M, N, K, 1.0, A, K, A, K, 0.0, C, N, 1, ws, cap,
              stream_ptr())
torch.cuda.synchronize()
print("ok")
