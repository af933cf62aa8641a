"""The NVLink all-reduce's CUDA-IPC path across two PROCESSES on one GPU
(distributed.P2PAllreduce: cudaMalloc'd symmetric buffers, IPC handles
exchanged, peers' buffers opened, csrc/skb_p2p.cu). The ranks' publish and
gather halves are ordered by the parent so no kernel ever waits on another
process's kernel (two waiting kernels on one GPU are not guaranteed to be
co-scheduled, B200_PROFILING.md); the timeout path is covered by
tests/test_gpu_p2p.py."""

import multiprocessing as mp

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

M = 3001
TMO = 4_000_000_000


def _worker(rank, conn):
    import sys
    from types import SimpleNamespace

    import torch as T
    sys.path.insert(0, conn.recv())
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200.distributed import P2PAllreduce
    from paper_2209_08722_b200.runtime import stream_ptr
    T.cuda.set_device(0)
    p2p = P2PAllreduce(SimpleNamespace(rank=rank, world=2), M)
    conn.send(p2p.alloc_local())
    p2p.open_peers(conn.recv())
    g = np.random.Generator(np.random.Philox(rank))
    while True:
        cmd = conn.recv()
        if cmd[0] == "quit":
            break
        _, epoch, mode = cmd
        x = T.from_numpy(g.standard_normal(M) if mode != 2 else np.zeros(M)).cuda()
        sent = x.cpu().numpy().copy()
        _lib.call("skb_p2p_allreduce", x, x, M, p2p.ld, rank, 2, p2p.data_ptrs.ctypes.data,
                  p2p.flag_ptrs.ctypes.data, epoch, mode, TMO, p2p.err, stream_ptr())
        T.cuda.synchronize()
        conn.send((sent, x.cpu().numpy(), int(p2p.err.item())))
    p2p.release()
    conn.send("bye")


def test_p2p_allreduce_over_cuda_ipc_two_processes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    ctx = mp.get_context("spawn")
    pipes, procs = [], []
    for r in range(2):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_worker, args=(r, b), daemon=True)
        p.start()
        a.send(root)
        pipes.append(a)
        procs.append(p)
    try:
        handles = [c.recv() for c in pipes]
        for c in pipes:
            c.send(handles)
        for epoch, (pub, gat) in enumerate([(1, 0), (0, 1), (1, 0)], start=1):
            pipes[pub].send(("run", epoch, 1))          # publish only: never waits
            sent_pub, _, err = pipes[pub].recv()
            assert err == 0
            pipes[gat].send(("run", epoch, 0))          # publish + gather (peer already there)
            sent_gat, out_gat, err = pipes[gat].recv()
            assert err == 0
            parts = {pub: sent_pub, gat: sent_gat}
            ref = parts[0] + parts[1]                   # rank order
            assert np.array_equal(out_gat, ref), epoch
            pipes[pub].send(("run", epoch, 2))          # the publisher gathers too
            _, out_pub, err = pipes[pub].recv()
            assert err == 0 and np.array_equal(out_pub, ref), epoch
        for c in pipes:
            c.send(("quit",))
            assert c.recv() == "bye"
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
