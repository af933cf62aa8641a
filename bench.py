"""Benchmark of the B200 hot path (BASELINE.json metric: A.D^2.A' matvec GB/s,
sketch-precond build ms, IPM time-to-solve) on configuration c2
(m = 1,000, n = 1,000,000 dense fp64 per GPU, CountSketch w = 4,000).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one fused A D^2 A' z pass (the PCG inner step, krylov_solvers.py:46-47)
over this rank's 8 GB column block. value = algorithmic bytes of all ranks per
step / max-over-ranks device time (weak scaling: each GPU holds a c2-size
block; N > 1 adds the NCCL allreduce of the m-vector the sharded math needs).
Extra keys: per-kernel roofline, e2e through the public API with host
buffers, sketch + preconditioner build time, a full IPM solve on the device,
and the CPU baseline (the oracle restatement of the reference's scipy path on
a bounded column sample).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M, N_PER_GPU, W_SKETCH = 1000, 1_000_000, 4000
# The solve uses the s = 4 sparse sign embedding (s = 1 CountSketch at
# w = 4m is a weak embedding whose PCG caps and v-retries stall the c2 trajectory).
METRIC = "A.D^2.A' matvec GB/s (fused single pass, fp64)"
CONFIG = {"workload": "c2: wide dense LP m=1000, n=1e6 per GPU (8 GB), fused A D^2 A' z "
                      "(PCG step)", "m": 1000, "n_per_gpu": 1_000_000, "global_batch": 1,
          "l2": "inputs larger than L2 (8 GB streamed per step)"}
S_SOLVE = 4  # s = 1 stalls at c2 (mu 6.7e-4 after 200 outer steps, measured); s = 4 converges


def algo_bytes(m: int, n: int) -> int:
    """Fused normal matvec: A once (8mn) + d2 (8n) + z in, u out (16m)."""
    return 8 * m * n + 8 * n + 16 * m


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU side


_CPU = {}


def _cpu_block(i):
    """Worker: the reference's NormalOperator.apply on one column block (fork-shared)."""
    op, z = _CPU["ops"][i], _CPU["z"]
    return op.apply(z)


class CpuNormalSample:
    """The reference's NormalOperator.apply (scipy CSR, krylov_solvers.py:46-47),
    restated in oracle/, on an m x n_s column sample of the c2 generator, using
    every host core: scipy's sparsetools hold the GIL, so the sample is split
    into one column block per forked worker process and the m-vector partials
    are summed (A D^2 A' z = sum_b A_b D_b^2 A_b' z)."""

    def __init__(self, m=M, n_s=100_000, procs=None):
        import multiprocessing as mp
        import scipy.sparse as sp
        from oracle import ipm_oracle as O
        self.m, self.n_s = m, n_s
        self.procs = max(1, procs or os.cpu_count() or 1)
        g = np.random.Generator(np.random.Philox(0))
        A = g.standard_normal((m, n_s))
        d = 10.0 ** g.uniform(-2, 2, n_s)
        z = g.standard_normal(m)
        blocks = np.array_split(np.arange(n_s), self.procs)
        _CPU["ops"] = [O.NormalOp(sp.csr_matrix(A[:, b]), d[b]) for b in blocks]
        _CPU["z"] = z
        self.pool = mp.get_context("fork").Pool(self.procs)

    def apply(self):
        return np.sum(self.pool.map(_cpu_block, range(self.procs)), axis=0)

    def close(self):
        self.pool.close()
        self.pool.join()

    def sample_text(self, reps):
        return (f"m={self.m}, n={self.n_s} column sample of c2 (A iid N(0,1) as scipy CSR, as "
                f"the reference stores it; oracle/ipm_oracle.py NormalOp restating "
                f"krylov_solvers.py:46-47), {self.procs} column blocks on {self.procs} worker "
                f"processes (sparsetools hold the GIL), {reps} applies")


def cpu_sample_normal(m=M, n_s=100_000, target_s=12.0, max_reps=20):
    """-> (GB/s, detail) of the all-core CPU baseline on a bounded sample."""
    cs = CpuNormalSample(m, n_s)
    try:
        cs.apply()
        times = []
        t_all = time.perf_counter()
        while len(times) < max_reps and (time.perf_counter() - t_all) < target_s:
            t0 = time.perf_counter()
            cs.apply()
            times.append(time.perf_counter() - t0)
    finally:
        cs.close()
    t = float(np.median(times))
    return algo_bytes(m, n_s) / t / 1e9, dict(reps=len(times), seconds_per_apply=t,
                                              cores=cs.procs,
                                              sample=cs.sample_text(f"median of {len(times)}"))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # bounded sample per step so K + W steps finish in a few minutes
    cs = CpuNormalSample()
    try:
        for _ in range(args.warmup):
            cs.apply()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            cs.apply()
        dt = (time.perf_counter() - t0) / args.steps
    finally:
        cs.close()
    val = algo_bytes(cs.m, cs.n_s) / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Philox, c2 generator)",
        "config": dict(CONFIG, n_sample_per_step=cs.n_s),
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": cs.procs,
                         "kind": "port", "sample": cs.sample_text(f"{args.steps} timed")},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU side


def run_ours(args):
    import torch
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200 import ipm_core as IC
    from paper_2209_08722_b200 import kernels as K
    from paper_2209_08722_b200 import preconditioning as PC
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.distributed import Comm
    from paper_2209_08722_b200.krylov_solvers import NormalOperator
    from paper_2209_08722_b200.lp_model import DeviceLP
    from paper_2209_08722_b200.runtime import F64, lda_for, stream_ptr, workspace

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    comm = Comm()
    m, n_loc = M, N_PER_GPU
    n = n_loc * world

    # ---- synthetic c2 block of this rank, generated in HBM (seeded per rank)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    cols = torch.zeros((n_loc, lda_for(m)), dtype=F64, device=dev)
    cols[:, :m].normal_(generator=gen)
    A = K.DeviceMatrix(cols, m)
    x0 = torch.rand(n_loc, dtype=F64, device=dev, generator=gen) + 0.5
    s0 = torch.rand(n_loc, dtype=F64, device=dev, generator=gen) + 0.5
    g0 = torch.Generator(device=dev)
    g0.manual_seed(7)
    y0 = torch.randn(m, dtype=F64, device=dev, generator=g0)
    b = torch.empty(m, dtype=F64, device=dev)
    K.gemv(A, x0, b)
    comm.allreduce_(b)
    c = torch.empty(n_loc, dtype=F64, device=dev)
    K.gemv_t(A, y0, c, add=s0)
    lp = DeviceLP.from_device(A, b, c, n, j0=rank * n_loc, comm=comm, name="c2_synthetic")
    d = torch.exp(torch.empty(n_loc, dtype=F64, device=dev).uniform_(-4.6, 4.6, generator=gen))
    op = NormalOperator(lp, d)
    z = torch.randn(m, dtype=F64, device=dev, generator=g0)
    u = torch.empty(m, dtype=F64, device=dev)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    per_rank_bytes = algo_bytes(m, n_loc)

    def timed(fn, k):
        comm.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        e1.synchronize()
        comm.barrier()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], dtype=F64, device=dev)
        comm.allreduce_(t, "max")
        return float(t.item())

    # ---- headline: fused normal matvec (colstream + fixed-order reduce [+ allreduce])
    step = lambda: op.apply(z, out=u)  # noqa: E731
    # clocks are sampled over the loaded window: headline, roofline and e2e loops
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    time.sleep(0.3)  # let the sampler start before the timed region
    ms = timed(step, args.steps)
    ms_step = ms / args.steps
    value = world * per_rank_bytes / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel alone (colstream pass, CUDA events on its stream)
    part = torch.empty(int(_lib.lib().skb_stream_workspace_bytes(m)) // 8 + 1, dtype=F64,
                       device=dev)
    npart = np.zeros(1, dtype=np.int32)

    def kstep():
        _lib.call("skb_normal_apply_partials", A.cols, m, A.n, A.lda, op._d2, z, part,
                  npart.ctypes.data, stream_ptr())

    for _ in range(args.warmup):
        kstep()
    kms = timed(kstep, args.steps) / args.steps
    peak, peak_src = peaks()
    achieved = per_rank_bytes / (kms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_colstream_normal.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "colstream_kernel<16,true,OpNormal> (skb_stream.cu)",
                "bytes_per_launch": per_rank_bytes, "ms_per_launch": round(kms, 4),
                "peak_source": peak_src}

    # ---- e2e: public API with host buffers (pinned z in, u out, every step)
    zh = torch.randn(m, dtype=F64, generator=torch.Generator().manual_seed(3)).pin_memory()
    uh = torch.empty(m, dtype=F64).pin_memory()
    zd = torch.empty(m, dtype=F64, device=dev)

    def e2e_step():
        zd.copy_(zh, non_blocking=True)
        op.apply(zd, out=u)
        uh.copy_(u, non_blocking=True)
        stream.synchronize()

    for _ in range(args.warmup):
        e2e_step()
    comm.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    comm.barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    tt = torch.tensor([e2e_s], dtype=F64, device=dev)
    comm.allreduce_(tt, "max")
    e2e_s = float(tt.item())
    e2e = {"value": round(world * per_rank_bytes / e2e_s / 1e9, 1), "unit": "GB/s",
           "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 8 * m,
           "api": "NormalOperator.apply (krylov_solvers.py), pinned host z -> u"}
    clk.__exit__(None, None, None)

    # ---- sketch + preconditioner build (hash K1, ADW K2, CholeskyQR2 K3) at w = 4000, s = 1
    rows = (lp.j0, lp.j0 + n_loc)
    build_ms = []
    parts_ms = {"hash": [], "sketch": [], "factor": []}
    for rep in range(max(2, min(args.steps, 5)) + 1):
        comm.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        W = S.build_sparse_embedding(n, W_SKETCH, 1, 12345 + rep, rows=rows)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X = S.apply_sketch(lp, d, W, check_positive=False)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        f = PC.build_preconditioner(X, sketch_tag=W.tag)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if rep == 0:
            continue  # warm-up
        build_ms.append((t3 - t0) * 1e3)
        parts_ms["hash"].append((t1 - t0) * 1e3)
        parts_ms["sketch"].append((t2 - t1) * 1e3)
        parts_ms["factor"].append((t3 - t2) * 1e3)
    sketch = {"ms": round(float(np.median(build_ms)), 3),
              "hash_ms": round(float(np.median(parts_ms["hash"])), 3),
              "adw_ms": round(float(np.median(parts_ms["sketch"])), 3),
              "factor_ms": round(float(np.median(parts_ms["factor"])), 3),
              "adw_GBps": round((8.0 * m * n_loc + 8 * n_loc + 8.0 * m * W_SKETCH) /
                                (np.median(parts_ms["sketch"]) * 1e-3) / 1e9, 1),
              "w": W_SKETCH, "s": 1}
    del X, f

    # ---- IPM time-to-solve (feasible start x0, y0, s0; gamma widened as in the reference)
    solve = None
    if not args.no_solve:
        try:
            start = IC.make_iterate(lp, x0, y0, s0)
            theta0 = start.min_xs / start.mu
            gamma = max(0.1, 1.0 - 0.999 * theta0)
            prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=W_SKETCH, s=S_SOLVE,
                               tol_outer=1e-8, seed=0)
            comm.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = IC.solve(lp, start, prm)
            torch.cuda.synchronize()
            secs = time.perf_counter() - t0
            solve = {"seconds": round(secs, 3), "outer": rep.outer, "sum_inner": rep.sum_inner,
                     "max_inner": rep.max_inner, "converged": rep.converged,
                     "mu_final": rep.mu_final, "objective": rep.objective,
                     "gamma_run": round(gamma, 6), "sigma": 0.5, "tol_outer": 1e-8,
                     "w": W_SKETCH, "s": S_SOLVE,
                     "ms_per_outer": round(secs * 1e3 / max(rep.outer, 1), 2)}
        except Exception as e:  # report, do not hide
            solve = {"error": f"{type(e).__name__}: {e}"}

    configs = None
    if world == 1 and not args.no_configs:
        del lp, op, A, cols, x0, s0, c, d, z, u, zd
        torch.cuda.empty_cache()
        try:
            configs = other_configs(dev)
        except Exception as e:  # report, do not hide
            configs = {"error": f"{type(e).__name__}: {e}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, det = cpu_sample_normal()
        cpu = {"value": round(v, 3), "unit": "GB/s", "cores": det["cores"], "kind": "port",
               "sample": det["sample"], "seconds_per_apply": round(det["seconds_per_apply"], 4)}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (A iid N(0,1) fp64 generated in HBM, seeded per rank)",
            "config": dict(CONFIG, n_total=n, parallelism=f"column-shard x{world}"),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
            "sketch_precond_build": sketch, "ipm_solve": solve,
            "other_configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def _ev_ms(fn, reps, torch):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def other_configs(dev):
    """Kernel-level numbers of BASELINE configs c3 / c4 / c5 at full size on this
    GPU (synthetic data of each config's shape in HBM; CUDA events after a
    warm-up): the fused normal matvec with its algorithmic GB/s, and the sketch
    + factor build. Full-size time-to-solve of these configs:
    profiles/r01_solve_c3_c4_c5.jsonl (tools/solve_configs.py)."""
    import torch
    from paper_2209_08722_b200 import kernels as K
    from paper_2209_08722_b200 import preconditioning as PC
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.lp_model import DeviceLP
    from paper_2209_08722_b200.runtime import F64, lda_for
    out = {}
    g = torch.Generator(device=dev)

    def build_ms(lp, d, n, w, s, kind):
        for rep in range(2):  # the first pass warms workspaces and allocations
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            W = (S.build_gaussian_sketch(n, w, 99 + rep) if kind == "gaussian"
                 else S.build_sparse_embedding(n, w, s, 99 + rep))
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            X = S.apply_sketch(lp, d, W, check_positive=False)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            PC.build_preconditioner(X)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            del W, X
        return [round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2), round((t3 - t2) * 1e3, 2)]

    # c3: dense m = 2000, n = 4e6 (64 GB)
    m, n = 2000, 4_000_000
    g.manual_seed(3)
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev)
    cols[:, :m].normal_(generator=g)
    A = K.DeviceMatrix(cols, m)
    d2 = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.5
    z = torch.randn(m, dtype=F64, device=dev, generator=g)
    u = torch.empty(m, dtype=F64, device=dev)
    ms = _ev_ms(lambda: K.normal_apply(A, d2, z, u), 5, torch)
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=dev),
                              torch.ones(n, dtype=F64, device=dev), n)
    b = build_ms(lp, d2.sqrt(), n, 8000, 1, "sparse")
    out["c3"] = {"m": m, "n": n, "matvec_ms": round(ms, 3),
                 "matvec_GBps": round((8.0 * m * n + 16 * n + 16 * m) / ms / 1e6, 1),
                 "sketch_w": 8000, "s": 1, "hash_adw_factor_ms": b}
    del A, cols, lp, d2
    torch.cuda.empty_cache()
    # c4: sparse m = 1e4, n = 2e7, 5 nnz / column (CSC)
    m, n, k = 10_000, 20_000_000, 5
    g.manual_seed(4)
    rows = torch.randint(0, m, (n, k), device=dev, generator=g, dtype=torch.int32)
    rows, _ = torch.sort(rows, dim=1)
    vals = torch.randn((n, k), dtype=F64, device=dev, generator=g)
    colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device=dev)
    A = K.SparseDeviceMatrix(colptr, rows.reshape(-1).contiguous(), vals.reshape(-1), m)
    del rows, vals
    d2 = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.5
    z = torch.randn(m, dtype=F64, device=dev, generator=g)
    u = torch.empty(m, dtype=F64, device=dev)
    ms = _ev_ms(lambda: K.normal_apply(A, d2, z, u), 5, torch)
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=dev),
                              torch.ones(n, dtype=F64, device=dev), n)
    b = build_ms(lp, d2.sqrt(), n, 40_000, 1, "sparse")
    nnz = n * k
    out["c4"] = {"m": m, "n": n, "nnz": nnz, "matvec_ms": round(ms, 3),
                 "matvec_GBps": round((12.0 * nnz + 16 * n + 16 * m) / ms / 1e6, 1),
                 "sketch_w": 40_000, "s": 1, "hash_adw_factor_ms": b}
    del A, lp, d2, colptr
    torch.cuda.empty_cache()
    # c5: A = diag(r) G, m = 1000, n = 2e6, dense Gaussian sketch w = 4000
    m, n, w = 1000, 2_000_000, 4000
    g.manual_seed(5)
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev)
    cols[:, :m].normal_(generator=g)
    A = K.DeviceMatrix(cols, m)
    d = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.5
    z = torch.randn(m, dtype=F64, device=dev, generator=g)
    u = torch.empty(m, dtype=F64, device=dev)
    ms = _ev_ms(lambda: K.normal_apply(A, d, z, u), 5, torch)
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=dev),
                              torch.ones(n, dtype=F64, device=dev), n)
    b = build_ms(lp, d, n, w, 0, "gaussian")
    out["c5"] = {"m": m, "n": n, "matvec_ms": round(ms, 3),
                 "matvec_GBps": round((8.0 * m * n + 16 * n + 16 * m) / ms / 1e6, 1),
                 "sketch": "gaussian", "sketch_w": w, "W_gen_adw_gemm_factor_ms": b,
                 "W_draws_per_s": round(n * w / (b[0] * 1e-3), 1),
                 "gemm_TFps": round(2.0 * m * n * w / (b[1] * 1e-3) / 1e12, 2)}
    del A, cols, lp
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the c3/c4/c5 kernel-level numbers (single-GPU runs only)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
