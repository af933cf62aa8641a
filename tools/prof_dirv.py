"""c2 directions pass + v-invariant product: fused (skb_directions_v) vs the two passes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200.runtime import F64, lda_for
m, n = int(os.environ.get("PROF_M", 1000)), int(os.environ.get("PROF_N", 1_000_000))
g = torch.Generator(device="cuda"); g.manual_seed(0)
cols = torch.randn((n, lda_for(m)), dtype=F64, device="cuda", generator=g)
A = K.DeviceMatrix(cols, m)
x = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.2
s = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.2
v = torch.randn(n, dtype=F64, device="cuda", generator=g) * 1e-3
dy = torch.randn(m, dtype=F64, device="cuda", generator=g)
e = lambda k: torch.empty(k, dtype=F64, device="cuda")
o = [e(n), e(n), e(m), e(n), e(m)]
def two():
    K.directions(A, dy, x, s, v, 0.1, o[0], o[1], o[2], atdy=o[3])
    K.gemv_ratio(A, v, s, o[4])
def fused():
    K.directions_v(A, dy, x, s, v, 0.1, o[0], o[1], o[2], o[4], atdy=o[3])
for name, fn in (("two passes", two), ("fused", fused)):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(10): fn()
    b.record(); b.synchronize()
    print(f"{name} ({os.environ.get('SKB_DIRV_ZSMEM', 'zreg')}): {a.elapsed_time(b) / 10:.3f} ms")
