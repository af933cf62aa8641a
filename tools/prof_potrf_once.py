"""One skb_potrf at Mp (env PROF_MP, default 1024) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
Mp = int(os.environ.get("PROF_MP", 1024))
g = np.random.Generator(np.random.Philox(Mp))
X = g.standard_normal((Mp + 64, Mp)); G = torch.from_numpy(np.tril(X.T @ X)).cuda()
st = torch.zeros(1, dtype=torch.int32, device="cuda")
ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, Mp + 64)))
_lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr()); torch.cuda.synchronize()
print("status", int(st.item()))
