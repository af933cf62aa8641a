"""Randomized sweep of skb_gemm with the INT8 emulation forced (SKB_GEMM_EMU=2)
against an 80-bit reference and the fp64-level bound (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKB_GEMM_EMU"] = "2"
import numpy as np
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200.runtime import stream_ptr, workspace

rng = np.random.default_rng(int(os.environ.get("FUZZ_SEED", 2)))
bad = 0
for case in range(int(os.environ.get("FUZZ_N", 40))):
    M, N = (int(v) for v in rng.integers(1, 1500, 2))
    K = int(rng.integers(256, 6000))
    ta, tb, low = (int(v) for v in rng.integers(0, 2, 3))
    if low:
        N = M
    alpha, beta = float(rng.standard_normal()), float(rng.choice([0.0, 1.0, -0.5]))
    opa = rng.standard_normal((M, K)) * np.exp(rng.uniform(-20, 20, (M, 1)))
    opb = rng.standard_normal((K, N)) * np.exp(rng.uniform(-20, 20, (1, N)))
    A = opa.T.copy() if ta else opa.copy()
    B = opb.T.copy() if tb else opb.copy()
    C0 = rng.standard_normal((M, N))
    Cd = torch.from_numpy(C0.copy()).cuda()
    c0 = _lib.lib().skb_gemm_ozaki_calls()
    ws, cap = workspace(int(_lib.lib().skb_gemm_ozaki_workspace_bytes(M, N, K)) + (64 << 20))
    _lib.call("skb_gemm", ta, tb, M, N, K, alpha, torch.from_numpy(A).cuda(), A.shape[1],
              torch.from_numpy(B).cuda(), B.shape[1], beta, Cd, N, low, 1, 0, 0, 0, ws, cap,
              stream_ptr())
    emu = _lib.lib().skb_gemm_ozaki_calls() - c0
    out = Cd.cpu().numpy()
    ref = alpha * (opa.astype(np.longdouble) @ opb.astype(np.longdouble)) + beta * C0
    ra = np.abs(opa).max(axis=1)[:, None]; cb = np.abs(opb).max(axis=0)[None, :]
    bnd = abs(alpha) * 2.0 ** -51 * (ra * np.abs(opb).sum(0)[None, :] + cb * np.abs(opa).sum(1)[:, None]) \
        + 2.0 ** -52 * np.abs(ref).astype(np.float64) + 1e-300
    mask = np.tril(np.ones((M, N), bool)) if low else np.ones((M, N), bool)
    err = np.abs(out - ref).astype(np.float64)
    ok = bool(np.all(err[mask] <= bnd[mask])) and emu == 1
    if low:
        ok = ok and np.array_equal(out[~mask], C0[~mask])
    bad += not ok
    print(f"case {case}: M={M} N={N} K={K} ta={ta} tb={tb} lower={low} beta={beta} emu={emu} ok={ok}"
          f" worst={float((err[mask] / bnd[mask]).max()) if mask.any() else 0:.3f}", flush=True)
print("FAILURES", bad)
sys.exit(1 if bad else 0)
