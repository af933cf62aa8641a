import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
Mp = 64
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((4 * Mp, Mp), dtype=torch.float64, device="cuda", generator=g)
spd = (X.t() @ X).contiguous()
G = spd.clone(); Li = torch.empty_like(spd)
ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, 4 * Mp)))
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    G.copy_(spd)
    _lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr())
    _lib.call("skb_trtri", G, Li, Mp, Mp, ws, cap, stream_ptr())
torch.cuda.synchronize()
