"""The NVLink one-shot all-reduce kernel (csrc/skb_p2p.cu) in one process on
one GPU: every "rank" gets its own symmetric buffers, and the ranks' publish /
gather halves run in an order in which no kernel waits on another (the
production mode 0 is used for the rank that gathers after all peers have
published). Sums are in rank order, identical on every rank; a peer that never
publishes makes the kernel time out to NaN instead of hanging."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


TMO = 4_000_000_000  # peer-flag timeout in SM cycles (~2 s)


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_08722_b200 import _lib
    return _lib


def _bufs(L, world, m):
    ld = m + (m & 1)
    nb = int(L.lib().skb_p2p_max_blocks(m))
    data = np.zeros(world, dtype=np.uint64)
    flags = np.zeros(world, dtype=np.uint64)
    for g in range(world):
        L.call("skb_p2p_alloc", 16 * ld, data[g:].ctypes.data)
        L.call("skb_p2p_alloc", 8 * nb, flags[g:].ctypes.data)
    return ld, data, flags


@pytest.mark.parametrize("world,m", [(2, 1000), (3, 10_000), (8, 777)])
def test_p2p_allreduce_rank_order(L, world, m):
    from paper_2209_08722_b200.runtime import stream_ptr
    ld, data, flags = _bufs(L, world, m)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = np.random.Generator(np.random.Philox(world * m))
    for epoch in range(1, 6):
        vs = [g.standard_normal(m) * 10.0 ** g.uniform(-3, 3) for _ in range(world)]
        ref = vs[0].copy()
        for v in vs[1:]:
            ref = ref + v  # rank order
        outs = [torch.from_numpy(v.copy()).cuda() for v in vs]
        gatherer = epoch % world
        for r in range(world):  # everyone else publishes first
            if r != gatherer:
                L.call("skb_p2p_allreduce", outs[r], outs[r], m, ld, r, world, data.ctypes.data,
                       flags.ctypes.data, epoch, 1, TMO, err, stream_ptr())
        L.call("skb_p2p_allreduce", outs[gatherer], outs[gatherer], m, ld, gatherer, world,
               data.ctypes.data, flags.ctypes.data, epoch, 0, TMO, err, stream_ptr())
        for r in range(world):
            if r != gatherer:
                L.call("skb_p2p_allreduce", outs[r], outs[r], m, ld, r, world, data.ctypes.data,
                       flags.ctypes.data, epoch, 2, TMO, err, stream_ptr())
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), ref)
    assert int(err.item()) == 0
    for p in list(data) + list(flags):
        L.call("skb_p2p_free", int(p))


def test_p2p_allreduce_times_out_instead_of_hanging(L):
    from paper_2209_08722_b200.runtime import stream_ptr
    m, world = 300, 2
    ld, data, flags = _bufs(L, world, m)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    x = torch.ones(m, dtype=torch.float64, device="cuda")
    # rank 0 gathers epoch 1 but rank 1 never publishes it
    # a short, configurable timeout (0.05 s of SM clock)
    L.call("skb_p2p_allreduce", x, x, m, ld, 0, world, data.ctypes.data, flags.ctypes.data, 1, 0,
           100_000_000, err, stream_ptr())
    torch.cuda.synchronize()
    assert int(err.item()) == 1 and torch.isnan(x).all()
    for p in list(data) + list(flags):
        L.call("skb_p2p_free", int(p))
