import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
os.environ["SKB_GEMM_EMU"] = "0"
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps * 1e3
h = 1024
ws, cap = workspace(1 << 28)
for ld in (10048, 10056, 10080):
    big = torch.randn((8 * h + h, ld), dtype=torch.float64, device="cuda")
    C = torch.empty((4, h, h), dtype=torch.float64, device="cuda")
    s = 2 * h * (ld + 1)
    f = lambda: _lib.call("skb_gemm", 0, 0, h, h, h, 1.0, big[h:], ld, big, ld, 0.0, C, h, 0, 4, s, s, h * h, ws, cap, stream_ptr())
    t = ev(f)
    print(f"ld={ld} batch4 h={h}: {t:.1f} us  {4*2*h**3/t/1e6:.1f} TF", flush=True)
    del big
big = torch.randn((4, 2 * h, h), dtype=torch.float64, device="cuda")
C = torch.empty((4, h, h), dtype=torch.float64, device="cuda")
f = lambda: _lib.call("skb_gemm", 0, 0, h, h, h, 1.0, big[:, h:], h, big, h, 0.0, C, h, 0, 4, 2 * h * h, 2 * h * h, h * h, ws, cap, stream_ptr())
t = ev(f)
print(f"contiguous batch4 h={h}: {t:.1f} us  {4*2*h**3/t/1e6:.1f} TF", flush=True)
