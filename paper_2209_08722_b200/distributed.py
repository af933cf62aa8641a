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

import torch

try:
    import torch.distributed as dist
except Exception:  # pragma: no cover
    dist = None

SUM, MAX, MIN = "sum", "max", "min"


class Comm:
    def __init__(self, group=None):
        self.group = group
        self.host_staging = False
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

    def allreduce_(self, t: torch.Tensor, op: str = SUM) -> torch.Tensor:
        if self.world > 1:
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
        """All-gather the per-rank slices of an n-vector into the full vector."""
        if self.world == 1:
            return t
        sizes = [shard_range(n, r, self.world) for r in range(self.world)]
        width = max(j1 - j0 for j0, j1 in sizes)
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

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)


def shard_range(n: int, rank: int, world: int):
    base, extra = divmod(n, world)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)
