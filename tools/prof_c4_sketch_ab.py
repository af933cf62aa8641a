"""A/B of the c4 CSC sketch kernels in one process (development aid):
row-sorting kernel (default) vs the bid-round kernel (SKB_CSC_SKETCH_BIDS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import solve_configs as SC
from paper_2209_08722_b200 import sketching as S
lp, x0, y0, s0, kw = SC.build("c4")
g = torch.Generator(device="cuda"); g.manual_seed(11)
d = torch.rand(lp.n, dtype=torch.float64, device="cuda", generator=g) + 0.5
for s in (4, 1):
    W = S.build_sparse_embedding(lp.n, 40000, s, 12345)
    res = {}
    for rep in range(3):
        for name in ("rows", "bids"):
            if name == "bids":
                os.environ["SKB_CSC_SKETCH_BIDS"] = "1"
            else:
                os.environ.pop("SKB_CSC_SKETCH_BIDS", None)
            X = S.apply_sketch(lp, d, W)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                X = S.apply_sketch(lp, d, W)
            b.record(); b.synchronize()
            res.setdefault(name, []).append(a.elapsed_time(b) / 5)
            if rep == 0:
                res[name + "_X"] = X.cols.clone()
    same = bool(torch.equal(res["rows_X"], res["bids_X"]))
    print(f"s={s}: rows {min(res['rows']):.2f} ms  bids {min(res['bids']):.2f} ms  identical={same}",
          flush=True)
    del res
