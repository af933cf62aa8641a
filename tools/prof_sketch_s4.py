"""c2 ADW at s = 4 (and s = 1): column-block mode vs per-bucket streaming (SKB_SKETCH_BLK=0)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_2209_08722_b200 import kernels as K, sketching as S  # noqa
from paper_2209_08722_b200.lp_model import DeviceLP  # noqa
from paper_2209_08722_b200.runtime import F64, lda_for  # noqa
m, n, w = 1000, 1_000_000, 4000
g = torch.Generator(device="cuda"); g.manual_seed(0)
cols = torch.zeros((n, lda_for(m)), dtype=F64, device="cuda"); cols[:, :m].normal_(generator=g)
A = K.DeviceMatrix(cols, m)
lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device="cuda"), torch.ones(n, dtype=F64, device="cuda"), n)
d = torch.rand(n, dtype=F64, device="cuda", generator=g) + 0.5
for s in (4, 1):
    W = S.build_sparse_embedding(n, w, s, 5)
    res = {}
    for mode in ("-1", "0"):
        os.environ["SKB_SKETCH_BLK"] = mode
        X = S.apply_sketch(lp, d, W, check_positive=False); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            X = S.apply_sketch(lp, d, W, check_positive=False)
        e1.record(); e1.synchronize()
        res[mode] = (e0.elapsed_time(e1) / 5, X.cols.clone())
    same = torch.equal(res["-1"][1], res["0"][1])
    print(f"s={s}: block mode {res['-1'][0]:.3f} ms, per-bucket {res['0'][0]:.3f} ms, identical {same}")
