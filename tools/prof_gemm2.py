import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import workspace, stream_ptr
ws, cap = workspace(1 << 28)
def ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps * 1e3
for (M, N, K, lower, ta, tb) in [(1000, 1000, 4000, 1, 1, 0), (1024, 1024, 4000, 0, 1, 0), (4000, 1000, 1024, 0, 0, 1),
                         (4096, 4096, 4096, 0, 0, 0), (4096, 4096, 4096, 0, 1, 1), (10000, 10000, 40000, 1, 1, 0),
                         (4000, 1000, 200000, 0, 1, 0)]:
    Am = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
    Bm = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda")
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    for mode in ("pipe", "old"):
        if mode == "old": os.environ["SKB_GEMM_NOPIPE"] = "1"
        else: os.environ.pop("SKB_GEMM_NOPIPE", None)
        us = ev(lambda: _lib.call("skb_gemm", ta, tb, M, N, K, 1.0, Am, Am.shape[1], Bm, Bm.shape[1], 0.0, C, N,
                              lower, 1, 0, 0, 0, ws, cap, stream_ptr()), reps=5 if K*M*N > 1e12 else 20)
        tf = 2.0 * M * N * K / (2 if lower else 1) / (us * 1e-6) / 1e12
        print(f"{mode} M={M} N={N} K={K} lower={lower} ta={ta} tb={tb}: {us:9.1f} us {tf:6.2f} TF/s", flush=True)
    oa = Am.t() if ta else Am
    ob = Bm.t() if tb else Bm
    tb_ = ev(lambda: torch.mm(oa, ob), reps=5)
    print(f"   torch {tb_:9.1f} us {2.0*M*N*K/(tb_*1e-6)/1e12:6.2f} TF/s", flush=True)
