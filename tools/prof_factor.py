"""Time the factor pieces on a c2-size sketch (w=4000, m=1000) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.kernels import DeviceMatrix
from paper_2209_08722_b200 import preconditioning as PC
from paper_2209_08722_b200.runtime import workspace, stream_ptr

m, w = int(os.environ.get("PROF_M", 1000)), int(os.environ.get("PROF_W", 4000))
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = DeviceMatrix(torch.randn((w, m + (m & 1)), dtype=torch.float64, device="cuda", generator=g), m)
Mp = int(_lib.lib().skb_factor_padded_dim(m))
G = torch.empty((Mp, Mp), dtype=torch.float64, device="cuda")
S = X.cols[:, :m]
ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(m, w)))
st = torch.zeros(1, dtype=torch.int32, device="cuda")
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps
def gram():
    _lib.call("skb_gemm", 1, 0, m, m, w, 1.0, X.cols, X.lda, X.cols, X.lda, 0.0, G, Mp, 1, 1, 0, 0, 0, ws, cap, stream_ptr())
print("gram (lower, K=w) ms", ev(gram))
spd = (S.t() @ S).contiguous()
def chol():
    G.zero_(); G[:m, :m].copy_(spd); G[m:, m:].fill_diagonal_(1.0)
    _lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr())
print("potrf (incl. copy) ms", ev(chol))
Li = torch.empty_like(G)
def tri():
    _lib.call("skb_trtri", G, Li, Mp, Mp, ws, cap, stream_ptr())
print("trtri ms", ev(tri))
Y = torch.empty_like(X.cols)
def ygemm():
    _lib.call("skb_gemm", 0, 1, w, m, m, 1.0, X.cols, X.lda, Li, Mp, 0.0, Y, X.lda, 0, 1, 0, 0, 0, ws, cap, stream_ptr())
print("Y = X Linv' ms", ev(ygemm))
print("full factor ms", ev(lambda: PC.build_preconditioner(X), reps=3))
f = PC.build_preconditioner(X)
Linv = torch.empty_like(G); LinvT = torch.empty_like(G)
stats = np.zeros(4)
def cq2():
    _lib.call("skb_factor_cholqr2", X.cols, X.lda, w, m, Linv, LinvT, None, stats.ctypes.data, ws, cap, stream_ptr())
print("skb_factor_cholqr2 alone ms", ev(cq2, reps=5))
print("rank_check alone ms", ev(lambda: PC.rank_check(f), reps=5))
