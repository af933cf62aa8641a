"""Column sharding across GPUs (one process per GPU, torch.distributed/NCCL).

A is split into contiguous column blocks; rank g holds columns [j0, j1) and
the matching slices of every n-vector (x, s, d, dx, ds, v, r_d). m-vectors
(y, dy, p, r_p, PCG vectors) and the factor are replicated. The only data
exchanges are the ones the math has:
  - every A-pass that produces an m-vector: allreduce-sum of the local sum;
  - the sketch ADW = sum_g A_g D_g W_g: allreduce-sum of the w x m partial;
  - scalar reductions of n-vectors (sums, max, min).
With world_size 1 every method is a no-op.
"""

from __future__ import annotations

import os

import torch

# Reproducible sharded parity: NCCL's sums are identical run to
# run only for a fixed rank count, message size and algorithm / protocol, so
# unless the user chose them (or SKB_NCCL_PIN=0) they are pinned here, before
# any communicator exists (import this package before init_process_group). The
# per-pass m-vector exchange does not go through NCCL at all (P2PAllreduce).
if os.environ.get("SKB_NCCL_PIN", "1") != "0":
    for _k, _v in (("NCCL_ALGO", "Ring"), ("NCCL_PROTO", "Simple")):
        os.environ.setdefault(_k, _v)

try:
    import torch.distributed as dist
except Exception:  # pragma: no cover
    dist = None

SUM, MAX, MIN = "sum", "max", "min"


class P2PAllreduce:
    """One-shot all-reduce of m-vectors over NVLink peer memory
    (csrc/skb_p2p.cu): symmetric buffers from cudaMalloc, opened by every peer
    through CUDA IPC; one kernel per all-reduce (publish, acquire the peers'
    flags, sum in rank order), no NCCL call on the per-pass path. Comm builds
    it collectively on the first eligible all-reduce, in phases that every rank
    agrees on before the next collective (so a local failure cannot leave a
    peer blocked), and checks it against NCCL once."""

    def __init__(self, comm: "Comm", cap: int):
        self.comm, self.rank, self.world = comm, comm.rank, comm.world
        self.ld = cap + (cap & 1)
        self.cap = cap
        self.epoch = 0
        self.err = None
        self._own = None
        self._opened = []
        self.data_ptrs = self.flag_ptrs = None

    def alloc_local(self):
        """Phase A (local): own buffers and their IPC handles (128 bytes)."""
        import numpy as np
        from . import _lib
        nb = int(_lib.lib().skb_p2p_max_blocks(self.cap))
        own = np.zeros(2, dtype=np.uint64)
        _lib.call("skb_p2p_alloc", 16 * self.ld, own[0:].ctypes.data)
        _lib.call("skb_p2p_alloc", 8 * max(nb, 1), own[1:].ctypes.data)
        self._own = own
        h = np.zeros(128, dtype=np.uint8)
        _lib.call("skb_ipc_handle", int(own[0]), h[:64].ctypes.data)
        _lib.call("skb_ipc_handle", int(own[1]), h[64:].ctypes.data)
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        return h

    def open_peers(self, handles):
        """Phase C (local): open every peer's buffers from the gathered handles."""
        import numpy as np
        from . import _lib
        self.data_ptrs = np.zeros(self.world, dtype=np.uint64)
        self.flag_ptrs = np.zeros(self.world, dtype=np.uint64)
        for g, hb in enumerate(handles):
            if g == self.rank:
                self.data_ptrs[g], self.flag_ptrs[g] = self._own[0], self._own[1]
                continue
            p = np.zeros(2, dtype=np.uint64)
            _lib.call("skb_ipc_open", hb[:64].ctypes.data, p[0:].ctypes.data)
            self._opened.append(int(p[0]))
            _lib.call("skb_ipc_open", hb[64:].ctypes.data, p[1:].ctypes.data)
            self._opened.append(int(p[1]))
            self.data_ptrs[g], self.flag_ptrs[g] = p[0], p[1]

    def release(self):
        from . import _lib
        for p in self._opened:
            try:
                _lib.call("skb_ipc_close", p)
            except Exception:
                pass
        self._opened = []

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        from . import _lib
        from .runtime import stream_ptr
        if t.numel() == 0:  # no launch: the epoch (slot parity) must not move
            return t
        self.epoch += 1
        _lib.call("skb_p2p_allreduce", t, t, t.numel(), self.ld, self.rank, self.world,
                  self.data_ptrs.ctypes.data, self.flag_ptrs.ctypes.data, self.epoch, 0,
                  p2p_timeout_cycles(), self.err, stream_ptr())
        return t

    def check(self):
        """Raise CollectiveTimeout if any exchange so far saw a peer time out
        (the kernel's sticky err word; one 4-byte read, done with the solve's
        per-step host scalars)."""
        if self.err is not None and int(self.err.item()) != 0:
            from .errors import CollectiveTimeout
            raise CollectiveTimeout(
                f"rank {self.rank}: a peer did not join an NVLink all-reduce within "
                f"{p2p_timeout_cycles()} SM cycles (epoch <= {self.epoch}); the exchanged "
                "m-vector was poisoned with NaN")


def p2p_timeout_cycles() -> int:
    """Peer-flag wait budget of the NVLink all-reduce in SM cycles:
    SKB_P2P_TIMEOUT_S seconds (default 2) at the B200's 1.965 GHz boost clock."""
    import os
    return max(1, int(float(os.environ.get("SKB_P2P_TIMEOUT_S", "2")) * 1.965e9))


def _p2p_enabled_env() -> bool:
    import os
    return os.environ.get("SKB_P2P", "1") != "0"


class Comm:
    def __init__(self, group=None):
        self.group = group
        self.host_staging = False
        self._p2p = None          # P2PAllreduce once built
        self._p2p_state = None    # None: not tried, False: unavailable
        if dist is not None and dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            # gloo (CPU tests, shared-GPU emulation) reduces through host copies
            self.host_staging = dist.get_backend(group) == "gloo"
        else:
            self.rank, self.world = 0, 1

    @property
    def active(self) -> bool:
        return self.world > 1

    def shard(self, n: int):
        """Balanced contiguous column range [j0, j1) of this rank."""
        return shard_range(n, self.rank, self.world)

    def _p2p_for(self, t: torch.Tensor):
        """The NVLink all-reduce for a float64 CUDA m-vector, built (collectively,
        on the first eligible call every rank makes with the same size) and
        checked against NCCL once; None where it does not apply."""
        if self._p2p_state is False or self.host_staging or not t.is_cuda:
            return None
        if t.dtype != torch.float64 or t.dim() != 1 or not t.is_contiguous():
            return None
        if self._p2p is not None:
            return self._p2p if t.numel() <= self._p2p.cap else None
        if not _p2p_enabled_env() or not (2 <= self.world <= 8):
            self._p2p_state = False
            return None
        if t.numel() > (1 << 17):  # m-vectors only (every rank sees the same sizes)
            return None
        from . import _lib
        dev_t = t.device
        ok = torch.ones(1, dtype=torch.float64, device=dev_t)

        def agree(flag: bool) -> bool:  # every rank learns whether all succeeded
            ok.fill_(1.0 if flag else 0.0)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
            return ok.item() == 1.0

        p2p = P2PAllreduce(self, max(t.numel(), 16384))
        h = None
        try:  # phase A (local): peer access to every rank's GPU, own buffers
            dev = torch.cuda.current_device()
            ids = [torch.zeros(1, dtype=torch.int64, device=dev_t) for _ in range(self.world)]
            dist.all_gather(ids, torch.tensor([dev], dtype=torch.int64, device=dev_t),
                            group=self.group)
            if all(_lib.lib().skb_p2p_can_access(dev, int(i.item())) for i in ids):
                h = p2p.alloc_local()
        except Exception:
            h = None
        if not agree(h is not None):
            self._p2p_state = False
            return None
        # phase B (collective): gather the handles
        ht = torch.from_numpy(h).to(dev_t)
        hs = [torch.empty_like(ht) for _ in range(self.world)]
        dist.all_gather(hs, ht, group=self.group)
        good = True
        try:  # phase C (local): open the peers' buffers
            p2p.open_peers([x.cpu().numpy() for x in hs])
        except Exception:
            good = False
        if agree(good):
            # phase D: one all-reduce checked against NCCL (a peer that never
            # arrives makes the kernel time out to NaN, never hang)
            g = torch.Generator(device=dev_t)
            g.manual_seed(1234 + self.rank)
            x = torch.randn(t.numel(), dtype=torch.float64, device=dev_t, generator=g)
            y = x.clone()
            p2p.allreduce_(x)
            dist.all_reduce(y, group=self.group)
            good = bool(torch.allclose(x, y, rtol=1e-12, atol=1e-12)) and \
                int(p2p.err.item()) == 0
            if agree(good):
                self._p2p, self._p2p_state = p2p, True
                return p2p
        p2p.release()
        self._p2p_state = False
        return None

    def allreduce_(self, t: torch.Tensor, op: str = SUM) -> torch.Tensor:
        if self.world > 1:
            if op == SUM:
                p2p = self._p2p_for(t)
                if p2p is not None:
                    return p2p.allreduce_(t)
            rop = {SUM: dist.ReduceOp.SUM, MAX: dist.ReduceOp.MAX, MIN: dist.ReduceOp.MIN}[op]
            if self.host_staging and t.is_cuda:
                h = t.cpu()
                dist.all_reduce(h, op=rop, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=rop, group=self.group)
        return t

    def combine_(self, vals: torch.Tensor, ops) -> torch.Tensor:
        """Combine a small vector of per-rank reduction results in place; ops[k]
        says how entry k combines (sum / max / min)."""
        if self.world == 1:
            return vals
        for kind in (SUM, MAX, MIN):
            idx = [k for k, o in enumerate(ops) if o == kind]
            if not idx:
                continue
            sel = torch.tensor(idx, device=vals.device)
            part = vals.index_select(0, sel).clone()
            self.allreduce_(part, kind)
            vals.index_copy_(0, sel, part)
        return vals

    def gather_columns(self, t: torch.Tensor, n: int) -> torch.Tensor:
        """All-gather the per-rank slices of an n-vector into the full vector
        (contiguous blocks in rank order, of any sizes: the phase-1 auxiliary LP
        puts its identity columns on the last rank)."""
        if self.world == 1:
            return t
        loc = torch.tensor([t.numel()], dtype=torch.int64,
                           device="cpu" if self.host_staging else t.device)
        lens = [torch.empty_like(loc) for _ in range(self.world)]
        dist.all_gather(lens, loc, group=self.group)
        lens = [int(v.item()) for v in lens]
        assert sum(lens) == n, (lens, n)
        sizes = []
        j = 0
        for ln in lens:
            sizes.append((j, j + ln))
            j += ln
        width = max(lens)
        dev = "cpu" if self.host_staging else t.device
        buf = torch.zeros(width, dtype=t.dtype, device=dev)
        buf[: t.numel()].copy_(t)
        out = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(out, buf, group=self.group)
        return torch.cat([o[: j1 - j0] for o, (j0, j1) in zip(out, sizes)]).to(t.device)

    def row_block(self, rows: int):
        """[r0, r1) of this rank's block when `rows` rows are scattered in equal
        chunks of ceil(rows / world) (the last ones may be short or empty)."""
        chunk = -(-rows // self.world)
        r0 = min(rows, self.rank * chunk)
        return r0, min(rows, r0 + chunk)

    def reduce_scatter_rows(self, X: torch.Tensor) -> torch.Tensor:
        """Sum X (rows x k, identical shape on every rank) over ranks and keep
        this rank's row block (row_block). One NCCL reduce-scatter (rows padded
        to a multiple of world); gloo sums on the host and slices."""
        rows = X.shape[0]
        r0, r1 = self.row_block(rows)
        if self.world == 1:
            return X
        if self.host_staging or not X.is_cuda:
            self.allreduce_(X)
            return X[r0:r1].contiguous()
        chunk = -(-rows // self.world)
        if chunk * self.world != rows:
            pad = torch.zeros((chunk * self.world - rows,) + tuple(X.shape[1:]), dtype=X.dtype,
                              device=X.device)
            X = torch.cat([X, pad])
        out = torch.empty((chunk,) + tuple(X.shape[1:]), dtype=X.dtype, device=X.device)
        dist.reduce_scatter_tensor(out, X.contiguous(), group=self.group)
        return out[: r1 - r0].contiguous()

    def allgather_rows(self, t: torch.Tensor, rows: int) -> torch.Tensor:
        """Inverse of the row-block split: every rank's block of a `rows`-long
        vector (or rows x k array) concatenated in rank order."""
        if self.world == 1:
            return t
        chunk = -(-rows // self.world)
        dev = "cpu" if self.host_staging else t.device
        buf = torch.zeros((chunk,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        buf[: t.shape[0]].copy_(t)
        out = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(out, buf, group=self.group)
        return torch.cat(out)[:rows].to(t.device)

    def all_to_all_v(self, t: torch.Tensor, send, recv) -> torch.Tensor:
        """1-D variable all-to-all: t holds this rank's pieces for ranks
        0..world-1 back to back (send[h] elements each); returns the pieces
        received from ranks 0..world-1 back to back (recv[h] each). NCCL
        all_to_all_single; over gloo every rank gathers every send buffer on
        the host and cuts its pieces out (tests and CPU runs)."""
        if self.world == 1:
            return t
        if not (self.host_staging or not t.is_cuda):
            out = torch.empty(sum(recv), dtype=t.dtype, device=t.device)
            dist.all_to_all_single(out, t, output_split_sizes=list(recv),
                                   input_split_sizes=list(send), group=self.group)
            return out
        sizes = torch.tensor(list(send), dtype=torch.int64)
        all_sizes = [torch.empty_like(sizes) for _ in range(self.world)]
        dist.all_gather(all_sizes, sizes, group=self.group)
        width = max(int(s.sum()) for s in all_sizes)
        buf = torch.zeros(max(width, 1), dtype=t.dtype)
        buf[: t.numel()].copy_(t.cpu())
        bufs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(bufs, buf, group=self.group)
        pieces = []
        for h in range(self.world):
            off = int(all_sizes[h][: self.rank].sum())
            pieces.append(bufs[h][off:off + int(all_sizes[h][self.rank])])
        return torch.cat(pieces).to(t.device)

    def check(self):
        """Surface an asynchronous exchange failure (CollectiveTimeout)."""
        if self._p2p is not None:
            self._p2p.check()

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)


def shard_range(n: int, rank: int, world: int):
    base, extra = divmod(n, world)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)
