"""Event-timed sketch apply at c2 (m=1000, n=1e6, w=4000) for s = 1, 4 (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200 import sketching as S
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for
m, n, w = 1000, int(os.environ.get("PROF_N", 1_000_000)), 4000
g = torch.Generator(device="cuda"); g.manual_seed(0)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device="cuda"); cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device="cuda"), torch.ones(n, dtype=F64, device="cuda"), n)
d = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.5
for s in (1, 4):
    W = S.build_sparse_embedding(n, w, s, 7)
    for _ in range(2): S.apply_sketch(lp, d, W, check_positive=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): S.apply_sketch(lp, d, W, check_positive=False)
    b.record(); b.synchronize()
    print(f"s={s}: {a.elapsed_time(b) / 5:.3f} ms (incl. bucket sort)")
