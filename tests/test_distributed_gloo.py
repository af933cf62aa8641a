"""Column-sharded host logic on world_size 2 over gloo (CPU): shard ranges,
the allreduce of per-rank m-vector partials, scalar combines (sum / max /
min) and the column gather used by the solve report."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2209_08722_b200.distributed import Comm
        comm = Comm()
        assert (comm.rank, comm.world) == (rank, world)
        m, n = 7, 1003
        g = np.random.default_rng(0)
        A = g.standard_normal((m, n))
        x = g.standard_normal(n)
        j0, j1 = comm.shard(n)
        # per-rank column-block partial of A x (what the streaming kernel returns)
        part = torch.from_numpy(A[:, j0:j1] @ x[j0:j1])
        comm.allreduce_(part)
        full = A @ x
        err = float(np.max(np.abs(part.numpy() - full)) / np.max(np.abs(full)))
        # scalar stats combine: sum, max, min in one call
        loc = x[j0:j1]
        st = torch.tensor([float((loc * loc).sum()), float(loc.max()), float(loc.min())],
                          dtype=torch.float64)
        comm.combine_(st, ("sum", "max", "min"))
        ok_stats = (abs(st[0].item() - float(x @ x)) <= 1e-12 * float(x @ x)
                    and st[1].item() == x.max() and st[2].item() == x.min())
        gathered = comm.gather_columns(torch.from_numpy(x[j0:j1].copy()), n).numpy()
        # distributed sketch: reduce-scatter of the w x m partial by bucket blocks,
        # Gram of the blocks summed, and the block vector gathered back (w = 11: uneven)
        w = 11
        Pall = np.random.default_rng(5).standard_normal((world, w, m))
        P = torch.from_numpy(Pall[rank].copy())
        total = Pall.sum(axis=0)
        r0, r1 = comm.row_block(w)
        blk = comm.reduce_scatter_rows(P.clone())
        ok_rs = blk.shape == (r1 - r0, m) and np.allclose(blk.numpy(), total[r0:r1], atol=1e-14)
        G = blk.T @ blk
        comm.allreduce_(G)
        ok_gram = np.allclose(G.numpy(), total.T @ total, rtol=1e-13, atol=1e-13)
        u = comm.allgather_rows(torch.arange(r0, r1, dtype=torch.float64), w)
        ok_ag = np.array_equal(u.numpy(), np.arange(w, dtype=np.float64))
        q.put((rank, err, ok_stats, bool(np.array_equal(gathered, x)), (j0, j1),
               ok_rs and ok_gram and ok_ag))
    finally:
        dist.destroy_process_group()


def test_sharded_host_logic_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][4] == (0, 502) and res[1][4] == (502, 1003)
    for _, err, ok_stats, ok_gather, _, ok_dist in res:
        assert err <= 1e-13 and ok_stats and ok_gather and ok_dist


def test_nccl_algorithm_pinned_for_reproducible_sums():
    """NCCL_ALGO / NCCL_PROTO pinned on import unless set."""
    import os
    import subprocess
    import sys
    code = ("import os; import paper_2209_08722_b200.distributed; "
            "print(os.environ['NCCL_ALGO'], os.environ['NCCL_PROTO'])")
    env = {k: v for k, v in os.environ.items() if k not in ("NCCL_ALGO", "NCCL_PROTO")}
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    out = subprocess.run([sys.executable, "-c", code], env=dict(env, PYTHONPATH=root),
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.stdout.split() == ["Ring", "Simple"], out.stderr
    out = subprocess.run([sys.executable, "-c", code],
                         env=dict(env, PYTHONPATH=root, NCCL_ALGO="Tree"),
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.stdout.split() == ["Tree", "Simple"], out.stderr
