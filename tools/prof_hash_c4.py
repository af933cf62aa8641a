import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2209_08722_b200 import sketching as S
n, w = 20_000_000, 40_000
for s in (1, 4):
    W = S.build_sparse_embedding(n, w, s, 1); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(5): W = S.build_sparse_embedding(n, w, s, 2 + r)
    torch.cuda.synchronize()
    print(f"s={s}: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms per build_sparse_embedding", flush=True)
