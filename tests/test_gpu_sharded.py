"""Column-sharded solve with real kernels: world size 2 on
one GPU, ranks exchanging through gloo (host-staged allreduce, no kernel
waits on another rank's kernel). Checks the whole sharded path -- hash slice,
partial-sketch allreduce, m-vector allreduces after every A-pass, scalar
combines, the gated PCG launch sequence, column gather -- against the
reference trajectory."""

import json
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q, kind="sparse"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2209_08722_b200 import ipm_core as IC
        from paper_2209_08722_b200.distributed import Comm
        from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
        from paper_2209_08722_b200.problems import wide_dense_lp
        comm = Comm()
        if kind == "sparse_csc":
            import scipy.sparse as sp
            from paper_2209_08722_b200.problems import sparse_wide_lp
            lpd = sparse_wide_lp(100, 20_000, 5, 7)
            dlp = DeviceLP.from_host(LinearProgram(sp.csr_matrix(lpd.A), lpd.b, lpd.c),
                                     comm=comm)
            assert dlp.sparse
        else:
            lpd = wide_dense_lp(40, 3000, 5)
            dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c), comm=comm)
        st = IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0)
        if kind == "sparse_csc":
            prm = IC.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=400, s=4,
                               tol_outer=1e-6, seed=11)
        elif kind == "gaussian":
            prm = IC.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5,
                               sketch="gaussian", w=160, tol_outer=1e-6, seed=9)
        else:
            prm = IC.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=160, s=4,
                               tol_outer=1e-7, seed=3)
        rep = IC.solve(dlp, st, prm)
        q.put((rank, rep.outer, [r.inner_iterations for r in rep.steps], rep.mu_trace,
               rep.objective, rep.x.shape[0], [r.sketch_seed for r in rep.steps], lpd.n))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "sparse"), (3, "sparse"), (2, "gaussian"),
                                        (2, "sparse_csc")])
def test_sharded_solve_matches_reference(world, kind):
    """Sharded sketch + distributed CholeskyQR2 (bucket-row blocks, Gram
    allreduce; world 3 gives uneven blocks) against the reference trajectory."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, kind))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] != "error" for r in res), res
    if kind == "gaussian":
        with open(os.path.join(GOLDEN, "gaussian_traces.json")) as f:
            gold = json.load(f)["wide"]
    elif kind == "sparse_csc":
        with open(os.path.join(GOLDEN, "sparse_traces.json")) as f:
            gold = json.load(f)["s4"]
    else:
        with open(os.path.join(GOLDEN, "small_traces.json")) as f:
            gold = json.load(f)["feasible"]
    for rank, outer, inner, mu, obj, nx, seeds, n_lp in res:
        assert outer == gold["outer"] and inner == gold["inner_iterations"]
        assert seeds == [s["sketch_seed"] for s in gold["steps"]]
        assert nx == n_lp
        dev = np.abs(np.array(mu) - np.array(gold["mu_trace"])) / np.array(gold["mu_trace"])
        # sharded sums change the summation order: the small LP's late steps amplify
        # any reordering of the reference itself to ~1.1e-8
        print(f"[{kind} rank {rank}] max mu rel dev {dev.max():.2e}, "
              f"objective rel dev {abs(obj - gold['objective']) / abs(gold['objective']):.2e}")
        assert dev.max() <= 5e-8, dev.max()
        assert abs(obj - gold["objective"]) <= 1e-8 * abs(gold["objective"])
    assert all(r[3] == res[0][3] for r in res)  # replicated scalars identical on every rank


def _start_rank(rank, world, port, q):
    """No-start feasible solve of a sparse LP, column-sharded: phase 1 with the
    identity columns on the last rank, PCG projection, shifted dual, centering."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2209_08722_b200 import ipm_core as IC
        from paper_2209_08722_b200.distributed import Comm
        from paper_2209_08722_b200.lp_model import DeviceLP
        from paper_2209_08722_b200.lp_model import random_feasible_lp as rfl
        dlp = DeviceLP.from_host(rfl(60, 4000, 0.02, 5), comm=Comm())
        prm = IC.IpmParams(mode="feasible", gamma=0.5, sigma=0.5, tol_outer=1e-6, seed=4)
        rep = IC.solve(dlp, None, prm)
        q.put((rank, rep.outer, [r.inner_iterations for r in rep.steps], rep.mu_trace,
               rep.objective, rep.x.shape[0]))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_solve_without_start_sparse():
    """SURVEY.md §8(f)2 under sharding: the whole start construction on a
    column-sharded sparse LP (world 2, gloo) against the reference's run."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    with open(os.path.join(GOLDEN, "start_sparse_traces.json")) as f:
        gs = json.load(f)["solve"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_start_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] != "error" for r in res), res
    for rank, outer, inner, mu, obj, nx in res:
        dev = np.max(np.abs(np.array(mu) - gs["mu_trace"]) / np.array(gs["mu_trace"]))
        print(f"[sharded start rank {rank}] outer {outer} (ref {gs['outer']}), "
              f"max mu rel dev {dev:.2e}")
        assert nx == 4000 and outer == gs["outer"] and inner == gs["inner_iterations"]
        assert dev <= 1e-6
        assert abs(obj - gs["objective"]) <= 1e-8 * abs(gs["objective"])


def _gauss_rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2209_08722_b200 import sketching as S
        from paper_2209_08722_b200.distributed import Comm
        comm = Comm()
        n, w = 20_011, 97
        rows = comm.shard(n)
        W = S.build_gaussian_sketch(n, w, 4242, rows=rows, comm=comm)
        q.put((rank, rows, W.dense.cpu().numpy()))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gaussian_w_stream_slices_bit_exact(world):
    """Rank-parallel W: each rank generates one slice of the Philox stream,
    draw offsets from the per-rank counts, one all-to-all for the draws that
    landed on a neighbour — identical to the single-device W (and to numpy)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from oracle import ipm_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_gauss_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] != "error" for r in res), res
    full = O.gaussian_sketch(20_011, 97, 4242)
    for rank, (j0, j1), blk in res:
        assert np.array_equal(blk, full[j0:j1]), rank


def _config_rank(rank, world, port, q, case):
    """A config-size instance (tests/golden/cfg_<case>.json) solved column-sharded."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2209_08722_b200 import ipm_core as IC
        from paper_2209_08722_b200.distributed import Comm
        from paper_2209_08722_b200.errors import MaxIterations
        from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
        from paper_2209_08722_b200.problems import wide_dense_lp
        with open(os.path.join(GOLDEN, f"cfg_{case}.json")) as f:
            g = json.load(f)
        kind, m, n, seed = g["gen"]
        if kind == "sparse":
            from paper_2209_08722_b200.problems import sparse_wide_lp
            lpd = sparse_wide_lp(m, n, 5, seed)
        else:
            lpd = wide_dense_lp(m, n, seed)
        dlp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c), comm=Comm())
        prm = IC.IpmParams(mode="feasible", gamma=g["gamma_run"], sigma=g["sigma"], w=g["w"],
                           s=4, tol_outer=g["tol_outer"], seed=g["seed"],
                           max_outer=g["steps_limit"] or 200)
        try:
            rep = IC.solve(dlp, IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0), prm)
        except MaxIterations as e:
            rep = e.report
        q.put((rank, rep.outer, [r.inner_iterations for r in rep.steps],
               [r.sketch_seed for r in rep.steps], [r.mu_after for r in rep.steps],
               [r.inner_residual_norms for r in rep.steps]))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["m2000", "sparse1e4"])
def test_sharded_config_size_vs_live_reference(case):
    """2000 x 1e5 (warp-pair streaming kernel, w = 8000) and the 1e4 x 2e5 CSC LP
    (w = 4e4: CSC sketch, INT8-emulated Grams) column-sharded over 2 ranks (gloo,
    one GPU): the distributed CholeskyQR2 and the m-vector all-reduces against
    the live reference's first steps -- same seeds and inner counts, mu and PCG
    residuals at the config gates of test_gpu_configs."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    path = os.path.join(GOLDEN, f"cfg_{case}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    import torch.multiprocessing as mp
    with open(path) as f:
        gold = json.load(f)["s4"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_config_rank, args=(r, 2, port, q, case)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] != "error" for r in res), res
    steps = gold["steps"]
    for rank, outer, inner, seeds, mu, rn in res:
        assert outer == gold["outer"]
        assert inner == [s["inner_iterations"] for s in steps]
        assert seeds == [s["sketch_seed"] for s in steps]
        dmu = max(abs(a - s["mu_after"]) / s["mu_after"] for a, s in zip(mu, steps))
        drn = max(float(np.max(np.abs(np.array(a) - np.array(s["inner_residual_norms"]))))
                  / s["f_norm0"] for a, s in zip(rn, steps))
        print(f"[sharded {case} rank {rank}] outer {outer}: mu {dmu:.2e}, residual/f0 {drn:.2e}")
        assert dmu <= 1e-9 and drn <= 1e-9
