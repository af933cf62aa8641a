"""Benchmark of the B200 hot path (BASELINE.json metric: A.D^2.A' matvec GB/s,
sketch-precond build ms, IPM time-to-solve).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4]

A "step" is one fused A D^2 A' z pass (the PCG inner step, krylov_solvers.py:46-47).
value = algorithmic bytes of all ranks per step / max-over-ranks device time.

Configs (BASELINE.json):
  c2 (default)  m = 1,000, n = 1e6 dense fp64 PER GPU (weak scaling). At N = 1 the
                data is the seeded SURVEY.md §8(d) generator (numpy Philox on the host,
                the instance tests/golden/cfg_c2.json recorded from the live
                reference); at N > 1 each rank generates its block in HBM.
  c3            m = 2,000, n = 4e6 dense (64 GB) split over N GPUs (strong scaling).
  c4            m = 1e4, n = 2e7, 5 nnz/column CSC (1e8 nnz) split over N GPUs (strong).

--gpus N without a torchrun environment launches N ranks itself
(torch.distributed.run, 127.0.0.1); every rank checks WORLD_SIZE == N.
Extra keys: per-kernel roofline, e2e through the public API with host buffers,
sketch + preconditioner build, a full IPM solve (c2: compared step by step with
the reference's own trace of the same instance), and the CPU baseline (the
oracle restatement of the reference's scipy path on every host core, at the
config's full size).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(m=1000, n=1_000_000, kind="dense", w=4000, scaling="weak",
               workload="c2: wide dense LP m=1000, n=1e6 per GPU (8 GB), fused A D^2 A' z "
                        "(PCG step)"),
    "c3": dict(m=2000, n=4_000_000, kind="dense", w=8000, scaling="strong",
               workload="c3: sharded wide dense LP m=2000, n=4e6 (64 GB) column-split over "
                        "the GPUs, fused A D^2 A' z + m-vector all-reduce"),
    "c4": dict(m=10_000, n=20_000_000, kind="sparse", k=5, w=40_000, scaling="strong",
               workload="c4: sparse wide LP m=1e4, n=2e7, 5 nnz/col CSC (1e8 nnz) column-split "
                        "over the GPUs, fused A D^2 A' z + m-vector all-reduce"),
}
METRIC = "A.D^2.A' matvec GB/s (fused single pass, fp64)"
S_SOLVE = 4  # s = 1 stalls at c2 (mu 6.7e-4 after 200 outer steps, measured); s = 4 converges


def algo_bytes(m: int, n: int, nnz: int | None = None) -> int:
    """Fused normal matvec, A read once: dense 8mn + 8n (d2) + 16m (z in, u out);
    CSC 12 nnz + 8(n+1) + 8n + 16m."""
    if nnz is None:
        return 8 * m * n + 8 * n + 16 * m
    return 12 * nnz + 8 * (n + 1) + 8 * n + 16 * m


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
#
# The reference's hot path on the host cores: oracle/ipm_oracle.py restates
# NormalOperator.apply (krylov_solvers.py:46-47: scipy csr_matvec + csc_matvec),
# apply_sketch (sketching.py:142-161: A.multiply(d) @ W as scipy csr_matmat)
# and build_preconditioner (preconditioning.py:38-51: LAPACK gesdd). scipy's
# sparsetools hold the GIL and are single-threaded, so the full-size A is split
# into one column block per worker PROCESS (each generates its own block) and
# the m-vector (m x w) partials are summed: A D^2 A' z = sum_b A_b D_b^2 A_b' z,
# ADW = sum_b A_b D_b W_b. The SVD runs in the parent on every BLAS thread.


def _cpu_worker(conn, m, nb, seed, kind, k):
    import scipy.sparse as sp
    from oracle import ipm_oracle as O
    g = np.random.Generator(np.random.Philox(seed))
    if kind == "dense":  # the reference's CSR storage, sharing the dense buffer
        dense = g.standard_normal((m, nb))
        A = sp.csr_matrix((dense.reshape(-1), np.tile(np.arange(nb, dtype=np.int32), m),
                           np.arange(0, m * nb + 1, nb, dtype=np.int64)), shape=(m, nb))
    else:
        rows = g.integers(0, m, size=(nb, k))
        rows.sort(axis=1)
        vals = g.standard_normal((nb, k))
        A = sp.csc_matrix((vals.ravel(), rows.ravel(), np.arange(0, nb * k + 1, k)),
                          shape=(m, nb)).tocsr()
    x = g.uniform(0.5, 1.5, nb)
    s = g.uniform(0.5, 1.5, nb)
    d = np.sqrt(x / s)
    op = O.NormalOp(A, d)
    conn.send(("ready", A.nnz))
    while True:
        msg = conn.recv()
        if msg[0] == "apply":
            conn.send(op.apply(msg[1]))
        elif msg[0] == "sketch":
            _, cols, vals, w = msg
            W = O.Sketch("sparse", nb, w, cols.shape[1], 0, cols=cols, vals=vals)
            conn.send(O.apply_sketch(A, d, W))
        else:
            break


class CpuPath:
    """The reference's CPU hot path over the whole config (see above)."""

    def __init__(self, m, n, kind="dense", k=5, procs=None, seed=0):
        import multiprocessing as mp
        self.m, self.n, self.kind = m, n, kind
        self.procs = max(1, procs or os.cpu_count() or 1)
        self.bounds = np.linspace(0, n, self.procs + 1).astype(np.int64)
        ctx = mp.get_context("fork")
        self.conns, self.ps = [], []
        for i in range(self.procs):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker, daemon=True,
                            args=(b, m, int(self.bounds[i + 1] - self.bounds[i]),
                                  seed * 1000 + i, kind, k))
            p.start()
            self.conns.append(a)
            self.ps.append(p)
        self.nnz = sum(a.recv()[1] for a in self.conns)
        self.z = np.random.Generator(np.random.Philox(seed + 7)).standard_normal(m)

    def apply(self):
        for a in self.conns:
            a.send(("apply", self.z))
        out = np.zeros(self.m)
        for a in self.conns:  # fixed order
            out += a.recv()
        return out

    def sketch_precond(self, w, s, seed):
        """(ms_hash, ms_adw, ms_svd): build_sparse_embedding on the parent (one
        sequential Philox stream), ADW over the workers, the SVD in the parent."""
        from oracle import ipm_oracle as O
        t0 = time.perf_counter()
        cols, vals = O.sparse_embedding(self.n, w, s, seed)
        t1 = time.perf_counter()
        for i, a in enumerate(self.conns):
            j0, j1 = self.bounds[i], self.bounds[i + 1]
            a.send(("sketch", cols[j0:j1], vals[j0:j1], w))
        adw = np.zeros((self.m, w))
        for a in self.conns:
            adw += a.recv()
        t2 = time.perf_counter()
        O.Factor(adw)
        t3 = time.perf_counter()
        return (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3

    def close(self):
        for a in self.conns:
            try:
                a.send(("quit",))
            except Exception:
                pass
        for p in self.ps:
            p.join(timeout=5)

    def bytes_per_apply(self):
        return algo_bytes(self.m, self.n, None if self.kind == "dense" else self.nnz)

    def sample_text(self, what):
        return (f"full config ({self.kind} m={self.m}, n={self.n}, nnz={self.nnz}) as scipy CSR, "
                f"as the reference stores it; oracle/ipm_oracle.py NormalOp restating "
                f"krylov_solvers.py:46-47, {self.procs} column blocks on {self.procs} worker "
                f"processes (sparsetools are single-threaded and hold the GIL), {what}")


def cpu_normal(cfg, target_s=10.0, max_reps=20, with_sketch=True):
    """-> (GB/s, detail dict) of the all-core CPU baseline at the config's full size."""
    c = CONFIGS[cfg]
    t_setup = time.perf_counter()
    cp = CpuPath(c["m"], c["n"], c["kind"], c.get("k", 5))
    setup_s = time.perf_counter() - t_setup
    try:
        cp.apply()
        times = []
        t_all = time.perf_counter()
        while len(times) < max_reps and (time.perf_counter() - t_all) < target_s:
            t0 = time.perf_counter()
            cp.apply()
            times.append(time.perf_counter() - t0)
        t = float(np.median(times))
        det = dict(reps=len(times), seconds_per_apply=t, cores=cp.procs, setup_s=setup_s,
                   sample=cp.sample_text(f"median of {len(times)} applies"))
        if with_sketch and c["kind"] == "dense":
            h, a, f = cp.sketch_precond(c["w"], 1, 12345)
            det["sketch_precond_build"] = {
                "ms": round(h + a + f, 1), "hash_ms": round(h, 1), "adw_ms": round(a, 1),
                "factor_ms": round(f, 1), "w": c["w"], "s": 1,
                "how": "oracle restatements of build_sparse_embedding (parent), apply_sketch "
                       "(sketching.py:142-161, column blocks on the workers) and the SVD of "
                       "build_preconditioner (preconditioning.py:38-51, parent, all BLAS "
                       "threads)"}
        return cp.bytes_per_apply() / t / 1e9, det
    finally:
        cp.close()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    c = dict(cfg)
    if args.config == "c3":
        # 8e9 nnz as scipy CSR is ~96 GB: more than a GPU box host holds alongside the
        # workers; the c3 CPU arm streams a 1/8 column block (the per-GPU share at N=8)
        c["n"] = cfg["n"] // 8
    cp = CpuPath(c["m"], c["n"], c["kind"], c.get("k", 5))
    try:
        for _ in range(args.warmup):
            cp.apply()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            cp.apply()
        dt = (time.perf_counter() - t0) / args.steps
    finally:
        cp.close()
    val = cp.bytes_per_apply() / dt / 1e9
    same = c["n"] == cfg["n"]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Philox per column block, the config's generator)",
        "config": {"workload": cfg["workload"], "m": c["m"], "n": c["n"],
                   "same_config": same, "global_batch": 1},
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": cp.procs,
                         "kind": "port", "sample": cp.sample_text(f"{args.steps} timed applies")},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU side


def _device_problem(cfg_name, world, rank, dev):
    """-> (DeviceLP, x0, y0, s0, d, source text, host LP or None) of this rank."""
    import torch

    from paper_2209_08722_b200 import kernels as K
    from paper_2209_08722_b200.distributed import Comm, shard_range
    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    from paper_2209_08722_b200.runtime import F64, lda_for
    c = CONFIGS[cfg_name]
    m = c["m"]
    comm = Comm()
    if cfg_name == "c2" and world == 1:
        from paper_2209_08722_b200.problems import wide_dense_lp
        t0 = time.perf_counter()
        lpd = wide_dense_lp(m, c["n"], 0)  # SURVEY.md §8(d), seed 0 (= tests/golden/cfg_c2)
        gen_s = time.perf_counter() - t0
        dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c, name=lpd.name))
        lpd.A = None
        x0 = torch.from_numpy(lpd.x0).to(dev)
        s0 = torch.from_numpy(lpd.s0).to(dev)
        y0 = torch.from_numpy(lpd.y0).to(dev)
        src = (f"SURVEY.md §8(d) generator wide_dense_lp(1000, 1e6, seed 0) on the host "
               f"(numpy Philox, {gen_s:.0f} s), uploaded")
        return dlp, x0, y0, s0, src, lpd
    n = c["n"] * world if c["scaling"] == "weak" else c["n"]
    j0, j1 = shard_range(n, rank, world)
    n_loc = j1 - j0
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    if c["kind"] == "dense":
        cols = torch.zeros((n_loc, lda_for(m)), dtype=F64, device=dev)
        cols[:, :m].normal_(generator=gen)
        A = K.DeviceMatrix(cols, m)
    else:
        k = c["k"]
        rows = torch.empty((n_loc, k), dtype=torch.int32, device=dev)
        # k distinct rows per column: k draws from disjoint strata of [0, m), then sorted
        base = torch.randint(0, m // k, (n_loc, k), device=dev, generator=gen, dtype=torch.int32)
        rows.copy_(base + torch.arange(k, device=dev, dtype=torch.int32) * (m // k))
        vals = torch.randn((n_loc, k), dtype=F64, device=dev, generator=gen)
        colptr = torch.arange(0, n_loc * k + 1, k, dtype=torch.int64, device=dev)
        A = K.SparseDeviceMatrix(colptr, rows.reshape(-1).contiguous(), vals.reshape(-1), m)
        del rows, vals, base
    x0 = torch.rand(n_loc, dtype=F64, device=dev, generator=gen) + 0.5
    s0 = torch.rand(n_loc, dtype=F64, device=dev, generator=gen) + 0.5
    g0 = torch.Generator(device=dev)
    g0.manual_seed(7)
    y0 = torch.randn(m, dtype=F64, device=dev, generator=g0)
    b = torch.empty(m, dtype=F64, device=dev)
    K.gemv(A, x0, b)
    comm.allreduce_(b)
    cvec = torch.empty(n_loc, dtype=F64, device=dev)
    K.gemv_t(A, y0, cvec, add=s0)
    dlp = DeviceLP.from_device(A, b, cvec, n, j0=j0, comm=comm, name=f"{cfg_name}_synthetic")
    src = (f"synthetic, generated in HBM per rank (torch Philox, seed 1000+rank): A iid N(0,1)"
           + ("" if c["kind"] == "dense" else f", {c['k']} distinct rows per column (strata)")
           + ", x0, s0 ~ U(0.5, 1.5), y0 ~ N(0,1), b = A x0, c = A'y0 + s0")
    return dlp, x0, y0, s0, src, None


def run_ours(args):
    import torch

    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200 import ipm_core as IC
    from paper_2209_08722_b200 import preconditioning as PC
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.krylov_solvers import NormalOperator
    from paper_2209_08722_b200.runtime import F64, stream_ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    dlp, x0, y0, s0, data_src, host_lp = _device_problem(args.config, world, rank, dev)
    comm = dlp.comm
    A = dlp.A
    m, n, n_loc = dlp.m, dlp.n, dlp.n_local
    sparse = dlp.sparse
    nnz_loc = int(A.vals.numel()) if sparse else None
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + rank)
    d = torch.exp(torch.empty(n_loc, dtype=F64, device=dev).uniform_(-4.6, 4.6, generator=gen))
    op = NormalOperator(dlp, d)
    g0 = torch.Generator(device=dev)
    g0.manual_seed(3)
    z = torch.randn(m, dtype=F64, device=dev, generator=g0)
    u = torch.empty(m, dtype=F64, device=dev)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    per_rank_bytes = algo_bytes(m, n_loc, nnz_loc)
    tot = torch.tensor([float(per_rank_bytes)], dtype=F64, device=dev)
    comm.allreduce_(tot)
    job_bytes = float(tot.item())

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

    # ---- headline: fused normal matvec (stream pass + fixed-order reduce [+ all-reduce])
    step = lambda: op.apply(z, out=u)  # noqa: E731
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    time.sleep(0.3)  # let the sampler start before the timed region
    ms = timed(step, args.steps)
    ms_step = ms / args.steps
    value = job_bytes / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel alone (CUDA events on its stream)
    peak, peak_src = peaks()
    if not sparse:
        part = torch.empty(int(_lib.lib().skb_stream_workspace_bytes(m)) // 8 + 1, dtype=F64,
                           device=dev)
        npart = np.zeros(1, dtype=np.int32)

        def kstep():
            _lib.call("skb_normal_apply_partials", A.cols, m, A.n, A.lda, op._d2, z, part,
                      npart.ctypes.data, stream_ptr())
        kname = "colstream_kernel<OpNormal> (skb_stream.cu)"
        prof = "ncu_colstream_normal.json"
    else:
        from paper_2209_08722_b200 import kernels as K

        def kstep():
            K.normal_apply(A, op._d2, z, u)
        kname = "csc normal pass + fixed-order reduce (skb_stream.cu)"
        prof = "ncu_csc_normal.json"
    for _ in range(args.warmup):
        kstep()
    kms = timed(kstep, args.steps) / args.steps
    achieved = per_rank_bytes / (kms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", prof)) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kname,
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
    e2e = {"value": round(job_bytes / e2e_s / 1e9, 1), "unit": "GB/s",
           "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": 8 * m,
           "api": "NormalOperator.apply (krylov_solvers.py), pinned host z -> u"}
    clk.__exit__(None, None, None)

    # ---- sketch + preconditioner build (hash K1, ADW K2, CholeskyQR2 K3)
    w_sk = cfg["w"]
    rows = (dlp.j0, dlp.j0 + n_loc)
    build = {}
    for s_nnz in (1, S_SOLVE):
        parts_ms = {"hash": [], "sketch": [], "factor": []}
        for rep in range(3):
            comm.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            W = S.build_sparse_embedding(n, w_sk, s_nnz, 12345 + rep, rows=rows)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            X = S.apply_sketch(dlp, d, W, check_positive=False)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            PC.build_preconditioner(X, sketch_tag=W.tag)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            if rep == 0:
                continue  # warm-up
            parts_ms["hash"].append((t1 - t0) * 1e3)
            parts_ms["sketch"].append((t2 - t1) * 1e3)
            parts_ms["factor"].append((t3 - t2) * 1e3)
            del X, W
        med = {k: float(np.median(v)) for k, v in parts_ms.items()}
        build[f"s{s_nnz}"] = {"ms": round(sum(med.values()), 3),
                              "hash_ms": round(med["hash"], 3),
                              "adw_ms": round(med["sketch"], 3),
                              "factor_ms": round(med["factor"], 3), "w": w_sk, "s": s_nnz}
    torch.cuda.empty_cache()

    # ---- IPM time-to-solve (feasible start x0, y0, s0; gamma widened as in the reference)
    solve = None
    if not args.no_solve:
        solve = _ipm_solve(IC, dlp, x0, y0, s0, cfg, host_lp, comm, torch)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del A, op
        try:
            v, det = cpu_normal(args.config)
            cpu = {"value": round(v, 3), "unit": "GB/s", "cores": det["cores"], "kind": "port",
                   "sample": det["sample"], "seconds_per_apply": round(det["seconds_per_apply"], 4),
                   "setup_s": round(det["setup_s"], 1)}
            if "sketch_precond_build" in det:
                cpu["sketch_precond_build"] = det["sketch_precond_build"]
            rec = _recorded_reference()
            if rec:
                cpu["reference_recorded"] = rec
        except Exception as e:  # report, do not hide
            cpu = {"error": f"{type(e).__name__}: {e}"[:300]}

    # ---- the other BASELINE configs on this GPU (kernel-level, synthetic data in HBM)
    other = None
    if world == 1 and args.config == "c2" and not args.no_other:
        other = {}
        try:
            del dlp
        except Exception:
            pass
        torch.cuda.empty_cache()
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs as BC
        for name in ("c3", "c4", "c5"):
            try:
                other[name] = getattr(BC, name)(1.0)
            except Exception as e:  # report, do not hide
                other[name] = {"error": f"{type(e).__name__}: {e}"[:200]}
            torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": data_src,
            "config": {"workload": cfg["workload"], "m": m, "n_total": n,
                       "n_per_gpu": n_loc, "global_batch": 1,
                       "l2": "inputs larger than L2 (A streamed from HBM every step)",
                       "parallelism": f"column-shard x{world}"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": 2 * args.steps * (1 if world == 1 else 2),
            "clocks": clk.summary(),
            "sketch_precond_build": build, "ipm_solve": solve,
        }
        if other is not None:
            line["other_configs"] = other
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def _recorded_reference():
    """The live reference's own c2 timings recorded in the build container
    (tests/golden/make_golden_configs.py, unmodified skipm on 8 cores)."""
    path = os.path.join(ROOT, "tests", "golden", "cfg_c2.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        g = json.load(f)
    out = {"host": f"build container, {g.get('host_cores')} cores, unmodified skipm "
                   "(tests/golden/make_golden_configs.py)"}
    for key in ("s4", "s1"):
        if key in g:
            out[f"seconds_per_outer_{key}"] = round(g[key]["seconds_per_outer"], 1)
    if "cpu_kernels" in g:
        out["kernels_s"] = {k: round(v, 3) for k, v in g["cpu_kernels"].items()
                            if k != "host_cores"}
    return out


def _ipm_solve(IC, dlp, x0, y0, s0, cfg, host_lp, comm, torch):
    try:
        start = IC.make_iterate(dlp, x0, y0, s0)
        theta0 = start.min_xs / start.mu
        gamma = max(0.1, 1.0 - 0.999 * theta0)
        prm = IC.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, w=cfg["w"], s=S_SOLVE,
                           tol_outer=1e-8, seed=0)
        comm.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = IC.solve(dlp, start, prm)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        out = {"seconds": round(secs, 3), "outer": rep.outer, "sum_inner": rep.sum_inner,
               "max_inner": rep.max_inner, "converged": rep.converged,
               "mu_final": rep.mu_final, "objective": rep.objective,
               "gamma_run": round(gamma, 6), "sigma": 0.5, "tol_outer": 1e-8,
               "w": cfg["w"], "s": S_SOLVE, "ms_per_outer": round(secs * 1e3 / max(rep.outer, 1), 2)}
        if host_lp is not None:
            out["vs_reference_trace"] = _vs_golden(rep)
        return out
    except Exception as e:  # report, do not hide
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def _vs_golden(rep):
    """The first outer steps of this solve against the live reference's trace of
    the same instance (tests/golden/cfg_c2.json, s = 4)."""
    path = os.path.join(ROOT, "tests", "golden", "cfg_c2.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        g = json.load(f).get("s4")
    if not g:
        return None
    k = len(g["steps"])
    st = rep.steps[:k]
    same = ([r.sketch_seed for r in st] == [s["sketch_seed"] for s in g["steps"]] and
            [r.inner_iterations for r in st] == [s["inner_iterations"] for s in g["steps"]])
    mu = max(abs(r.mu_after - s["mu_after"]) / s["mu_after"] for r, s in zip(st, g["steps"]))
    rn = max(float(np.max(np.abs(np.array(r.inner_residual_norms) -
                                 np.array(s["inner_residual_norms"])))) / s["f_norm0"]
             for r, s in zip(st, g["steps"]))
    return {"steps_compared": k, "seeds_and_inner_counts_identical": bool(same),
            "max_mu_rel_dev": mu, "max_residual_dev_over_f0": rn}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(argv, n):
    """Launch this script on n ranks (one process per GPU) when no torchrun
    environment is present."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def run_cpu_harness(args):
    """Harness check without a GPU (tests/test_bench_contract.py): the rank
    launch, barrier and max-over-ranks timing and the JSON line over gloo; a
    "step" is a host matvec standing in for the device pass."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        dist.init_process_group("gloo")
    a = torch.randn(256, 4096, dtype=torch.float64)
    z = torch.randn(256, dtype=torch.float64)
    for _ in range(args.warmup):
        a @ (a.t() @ z)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a @ (a.t() @ z)
    dt = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": "cpu harness check", "value": 1.0 / float(dt),
                          "unit": "steps/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": float(dt) * 1e3}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-other", action="store_true",
                    help="skip the c3 / c4 / c5 kernel timings of the default c2 run")
    ap.add_argument("--cpu-harness", action="store_true",
                    help="test mode: exercise the multi-rank harness over gloo without a GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(sys.argv[1:], args.gpus)
    if args.cpu_harness:
        return run_cpu_harness(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
