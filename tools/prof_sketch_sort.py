"""Dense sketch apply at c2 / c3 shapes (s = 4) with the counting or the radix
bucket order (SKB_BUCKET_RADIX / SKB_BUCKET_COUNTING), CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import kernels as K, sketching as S
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for
for (m, n, w) in [(1000, 1_000_000, 4000), (2000, 4_000_000, 8000)]:
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device="cuda"); cols[:, :m].normal_(generator=g)
    A = K.DeviceMatrix(cols, m)
    b = torch.zeros(m, dtype=F64, device="cuda"); c = torch.ones(n, dtype=F64, device="cuda")
    lp = DeviceLP.from_device(A, b, c, n)
    d = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.5
    W = S.build_sparse_embedding(n, w, 4, 7)
    X = S.apply_sketch(lp, d, W); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        X = S.apply_sketch(lp, d, W)
    e1.record(); e1.synchronize()
    print(f"m={m} n={n} w={w} s=4: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
    del cols, A, lp, X, W; torch.cuda.empty_cache()
