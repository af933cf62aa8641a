"""c4 CSC sketch apply (w = 4e4, s = 4 as in the solve) timing (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import solve_configs as SC
from paper_2209_08722_b200 import sketching as S
lp, x0, y0, s0, kw = SC.build("c4")
g = torch.Generator(device="cuda"); g.manual_seed(11)
d = torch.rand(lp.n, dtype=torch.float64, device="cuda", generator=g) + 0.5
s = int(os.environ.get("PROF_S", 4))
W = S.build_sparse_embedding(lp.n, 40000, s, 12345)
X = S.apply_sketch(lp, d, W)
torch.cuda.synchronize()
ref = X.cols.clone()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    X = S.apply_sketch(lp, d, W)
b.record(); b.synchronize()
print(f"c4 sketch apply s={s}: {a.elapsed_time(b) / 3:.2f} ms; bit-identical rerun:",
      bool(torch.equal(X.cols, ref)))
import hashlib
print("sha", hashlib.sha256(X.cols.cpu().numpy().tobytes()).hexdigest()[:16])
