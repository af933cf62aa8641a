"""skb_potrf timing vs Mp for the fused-step and the panel-loop paths (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
for Mp in (64, 128, 256, 512, 1024, 2048):
    g = np.random.Generator(np.random.Philox(Mp))
    X = g.standard_normal((Mp + 64, Mp)); S = torch.from_numpy(np.tril(X.T @ X)).cuda()
    G = S.clone(); st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, Mp + 64)))
    res = []
    for loop in ("0", "1"):
        os.environ["SKB_POTRF_LOOP"] = loop
        def run():
            G.copy_(S); _lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr())
        run(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): run()
        b.record(); b.synchronize(); res.append(a.elapsed_time(b) / 20 * 1e3)
    print(f"Mp {Mp:5d}: fused {res[0]:8.1f} us   loop {res[1]:8.1f} us", flush=True)
