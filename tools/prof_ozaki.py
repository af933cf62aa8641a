"""DMMA vs INT8-emulated FP64 GEMM on the factor / Gaussian-sketch shapes, and the
full CholeskyQR2 factor with the emulation on and off (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.kernels import DeviceMatrix
from paper_2209_08722_b200 import preconditioning as PC
from paper_2209_08722_b200.runtime import workspace, stream_ptr

L = _lib.lib()


def ev(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps


g = torch.Generator(device="cuda"); g.manual_seed(0)
shapes = [("gram c4", 1, 0, 10000, 10000, 40000, 1), ("Y c4", 0, 1, 40000, 10000, 10000, 0),
          ("gram c3", 1, 0, 2000, 2000, 8000, 1), ("c5 AdW", 1, 0, 4000, 1000, 2000000, 0),
          ("gram c2", 1, 0, 1000, 1000, 4000, 1)]
for name, ta, tb, M, N, K, low in shapes:
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda", generator=g)
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    lda, ldb = A.shape[1], B.shape[1]
    ws, cap = workspace(max(int(L.skb_gemm_ozaki_workspace_bytes(M, N, min(K, 65536))),
                            8 * 8 * M * N) + (64 << 20))
    os.environ["SKB_GEMM_EMU"] = "0"
    td = ev(lambda: _lib.call("skb_gemm", ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.0, C, N, low, 1,
                              0, 0, 0, ws, cap, stream_ptr()))
    Cd = C.clone()
    te = ev(lambda: _lib.call("skb_gemm_ozaki", ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.0, C, N,
                              low, ws, cap, stream_ptr()))
    if low:
        Cd, C = torch.tril(Cd), torch.tril(C)
    rel = float((C - Cd).abs().max() / Cd.abs().max())
    fl = 2.0 * M * N * K * (0.5 if low else 1.0)
    print(f"{name:8s} M={M} N={N} K={K}: dmma {td:8.2f} ms ({fl / td / 1e9:5.1f} TF)  "
          f"emu {te:8.2f} ms ({fl / te / 1e9:6.1f} TF-equiv)  x{td / te:4.2f}  maxrel {rel:.1e}",
          flush=True)
    del A, B, C, Cd, ws
    torch.cuda.empty_cache()

for m, w in [(2000, 8000), (10000, 40000)]:
    X = DeviceMatrix(torch.randn((w, m), dtype=torch.float64, device="cuda", generator=g), m)
    res = {}
    for mode in ("0", "1"):
        os.environ["SKB_GEMM_EMU"] = mode
        c0 = L.skb_gemm_ozaki_calls()
        t = ev(lambda: PC.build_preconditioner(X), reps=2)
        f = PC.build_preconditioner(X)
        res[mode] = f
        print(f"factor m={m} w={w} EMU={mode}: {t:.1f} ms, emulated GEMMs/call "
              f"{(L.skb_gemm_ozaki_calls() - c0) / 4:.0f}", flush=True)
    a, b = res["0"], res["1"]
    for attr in ("Linv",):
        x, y = getattr(a, attr, None), getattr(b, attr, None)
        if x is not None:
            print("  Linv maxrel diff", float((x - y).abs().max() / x.abs().max()))
    del X, res, a, b
    torch.cuda.empty_cache()
