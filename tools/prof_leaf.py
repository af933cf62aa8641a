"""Warm per-launch time of the potrf leaf (Mp = 64: one diagonal block) and of
skb_potrf / skb_trtri at a few Mp (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr

def ev(fn, reps=50):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps * 1e3

for Mp in [int(v) for v in os.environ.get("PROF_MPS", "64,128,256,1024,2048").split(",")]:
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    X = torch.randn((4 * Mp, Mp), dtype=torch.float64, device="cuda", generator=g)
    spd = (X.t() @ X).contiguous()
    G = torch.empty_like(spd); Li = torch.empty_like(spd)
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, 4 * Mp)))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    def potrf():
        G.copy_(spd)
        _lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr())
    def trtri():
        _lib.call("skb_trtri", G, Li, Mp, Mp, ws, cap, stream_ptr())
    copy = ev(lambda: G.copy_(spd))
    tp = ev(potrf) - copy
    tt = ev(trtri)
    err = (Li @ G - torch.eye(Mp, dtype=torch.float64, device="cuda")).abs().max().item()
    print(f"Mp={Mp:5d}: potrf {tp:8.1f} us  trtri {tt:8.1f} us  |Li L - I| {err:.1e}  status {int(st.item())}", flush=True)
