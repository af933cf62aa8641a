import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200 import sketching as S
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for
m, n = 2000, 4_000_000
g = torch.Generator(device="cuda"); g.manual_seed(3)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device="cuda"); cols[:, :m].normal_(generator=g)
lp = DeviceLP.from_device(K.DeviceMatrix(cols, m), torch.zeros(m, dtype=F64, device="cuda"), torch.ones(n, dtype=F64, device="cuda"), n)
d = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.5
for s in (1, 4):
    W = S.build_sparse_embedding(n, 8000, s, 11)
    X = S.apply_sketch(lp, d, W); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): X = S.apply_sketch(lp, d, W)
    b.record(); b.synchronize()
    print(f"c3 ADW s={s}: {a.elapsed_time(b) / 3:.2f} ms")
