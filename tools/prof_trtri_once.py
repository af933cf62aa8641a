"""One skb_trtri at Mp (PROF_MP) between cudaProfilerStart/Stop (launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
Mp = int(os.environ.get("PROF_MP", 10048))
g = torch.Generator(device="cuda"); g.manual_seed(0)
L = torch.tril(torch.randn((Mp, Mp), dtype=torch.float64, device="cuda", generator=g)) * 0.01
L += torch.eye(Mp, dtype=torch.float64, device="cuda") * 3
Li = torch.empty_like(L)
ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, 4 * Mp)))
_lib.call("skb_trtri", L, Li, Mp, Mp, ws, cap, stream_ptr()); torch.cuda.synchronize()
torch.cuda.profiler.start()
_lib.call("skb_trtri", L, Li, Mp, Mp, ws, cap, stream_ptr()); torch.cuda.synchronize()
torch.cuda.profiler.stop()
