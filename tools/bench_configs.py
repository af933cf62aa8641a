"""Per-config kernel timings on one B200 for the BASELINE configs beyond c2
(c3 dense m=2000, c4 sparse 1e8 nnz, c5 Gaussian sketch). Synthetic data in
HBM; CUDA-event timing after warm-up. Prints one JSON object per config.

    python tools/bench_configs.py [c3] [c4] [c5] [--scale S]

--scale shrinks n (per-kernel GB/s and TF/s are size-independent once the
operands exceed L2); the c3 64 GB and c5 64 GB W fit one B200 at scale 1.
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_08722_b200 import _lib  # noqa: E402
from paper_2209_08722_b200 import kernels as K  # noqa: E402
from paper_2209_08722_b200 import preconditioning as PC  # noqa: E402
from paper_2209_08722_b200 import sketching as S  # noqa: E402
from paper_2209_08722_b200.lp_model import DeviceLP  # noqa: E402
from paper_2209_08722_b200.runtime import F64, lda_for  # noqa: E402

DEV = torch.device("cuda")
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as _f:
        HBM_PEAK = float(json.load(_f)["hbm_gbs"])
except Exception:  # the profiling recipe's fallback
    HBM_PEAK = 7672.0


def ev(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def build_times(lp, d, n, w, s, kind="sparse", reps=2):
    out = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        W = (S.build_sparse_embedding(n, w, s, 500 + r) if kind == "sparse"
             else S.build_gaussian_sketch(n, w, 500 + r))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X = S.apply_sketch(lp, d, W, check_positive=False)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        PC.build_preconditioner(X)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if r:
            out.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))
        del W, X
    return [round(float(np.median([o[i] for o in out])), 3) for i in range(3)]


def c3(scale):
    m, n = 2000, int(4_000_000 * scale)
    g = torch.Generator(device=DEV)
    g.manual_seed(3)
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=DEV)
    cols[:, :m].normal_(generator=g)
    A = K.DeviceMatrix(cols, m)
    d2 = torch.rand(n, dtype=F64, device=DEV, generator=g) + 0.5
    z = torch.randn(m, dtype=F64, device=DEV, generator=g)
    u = torch.empty(m, dtype=F64, device=DEV)
    ms = ev(lambda: K.normal_apply(A, d2, z, u))
    byts = 8.0 * m * n + 8 * n + 16 * m
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=DEV),
                              torch.ones(n, dtype=F64, device=DEV), n)
    h, a, f = build_times(lp, d2.sqrt(), n, 8000, 1)
    return {"config": "c3 dense m=2000", "n": n, "matvec_ms": round(ms, 4),
            "matvec_GBps": round(byts / ms / 1e6, 1),
            "matvec_frac": round(byts / ms / 1e6 / HBM_PEAK, 3), "sketch_w": 8000, "hash_ms": h,
            "adw_ms": a, "factor_ms": f}


def c4(scale):
    m, n, k = 10_000, int(20_000_000 * scale), 5
    g = torch.Generator(device=DEV)
    g.manual_seed(4)
    rows = torch.randint(0, m, (n, k), device=DEV, generator=g, dtype=torch.int32)
    rows, _ = torch.sort(rows, dim=1)
    vals = torch.randn((n, k), dtype=F64, device=DEV, generator=g)
    colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device=DEV)
    A = K.SparseDeviceMatrix(colptr, rows.reshape(-1).contiguous(), vals.reshape(-1), m)
    d2 = torch.rand(n, dtype=F64, device=DEV, generator=g) + 0.5
    z = torch.randn(m, dtype=F64, device=DEV, generator=g)
    u = torch.empty(m, dtype=F64, device=DEV)
    ms = ev(lambda: K.normal_apply(A, d2, z, u))
    nnz = n * k
    byts = 12.0 * nnz + 8 * (n + 1) + 8 * n + 16 * m
    res = {"config": "c4 sparse m=1e4, 5 nnz/col", "n": n, "nnz": nnz,
           "matvec_ms": round(ms, 4), "matvec_GBps": round(byts / ms / 1e6, 1),
           "matvec_frac": round(byts / ms / 1e6 / HBM_PEAK, 3)}
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=DEV),
                              torch.ones(n, dtype=F64, device=DEV), n)
    h, a, f = build_times(lp, d2.sqrt(), n, 40_000, 1, reps=1)
    res.update(sketch_w=40_000, hash_ms=h, adw_ms=a, factor_ms=f)
    return res


def c5(scale):
    m, n, w = 1000, int(2_000_000 * scale), 4000
    g = torch.Generator(device=DEV)
    g.manual_seed(5)
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=DEV)
    cols[:, :m].normal_(generator=g)
    A = K.DeviceMatrix(cols, m)
    d = torch.rand(n, dtype=F64, device=DEV, generator=g) + 0.5
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=DEV),
                              torch.ones(n, dtype=F64, device=DEV), n)
    h, a, f = build_times(lp, d, n, w, 0, kind="gaussian", reps=1)
    flops = 2.0 * m * n * w
    return {"config": "c5 Gaussian sketch w=4000", "n": n, "W_gen_ms": h, "gemm_ms": a,
            "gemm_TFps": round(flops / (a * 1e-3) / 1e12, 2), "factor_ms": f,
            "W_draws_per_s": round(n * w / (h * 1e-3), 1)}


if __name__ == "__main__":
    args = sys.argv[1:]
    scale = 1.0
    if "--scale" in args:
        scale = float(args[args.index("--scale") + 1])
    todo = [a for a in args if a in ("c3", "c4", "c5")] or ["c3", "c4", "c5"]
    for name in todo:
        print(json.dumps(globals()[name](scale)), flush=True)
        torch.cuda.empty_cache()
