"""Sketch operators W and ADW on the device (reference sketching.py).

build_sparse_embedding draws the bucket/sign hashes on the GPU, bit-exact with
numpy's Philox stream (K1, csrc/skb_hash.cu); apply_sketch forms
X = (A diag(d) W)' bucket-major, bit-exact with scipy's csr_matmat order
(K2, csrc/skb_sketch.cu). Under column sharding every rank regenerates the
whole hash stream (the Lemire compaction needs the global prefix), keeps its
column slice, and the w x m partial sketches are allreduced.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .errors import DimensionMismatch, InvalidDims, NonpositiveScaling
from .runtime import F64, lda_for, require_cuda, stream_ptr, workspace


# Sharded runs keep ADW' distributed by bucket blocks and build the factor from
# the blocks (Gram allreduce) instead of allreducing the whole w x m sketch and
# factoring it on every rank.
DISTRIBUTED_FACTOR = True


def philox_key(seed: int):
    """numpy Philox(seed) key = SeedSequence(seed).generate_state(2, uint64)."""
    k = np.random.SeedSequence(int(seed)).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


@dataclass
class SketchOperator:
    """n x w sketch (reference SketchOperator, sketching.py:31-80).

    For kind "sparse_sign", cols/vals are device tensors holding the s
    buckets and values of this rank's rows [j0, j0 + n_local)."""

    kind: str
    n: int
    w: int
    s: int
    seed: int
    cols: torch.Tensor | None = None
    vals: torch.Tensor | None = None
    dense: torch.Tensor | None = None
    j0: int = 0
    words_used: int = 0

    @property
    def tag(self) -> tuple:
        return (self.kind, self.n, self.w, self.s, self.seed)

    def as_sparse(self):
        """W (this rank's rows) as a host scipy CSR matrix with sorted column
        indices (sketching.py:53-69); identity and sparse-sign sketches only."""
        import scipy.sparse as sp
        if self.kind == "identity":
            return sp.identity(self.n, format="csr")[self.j0:self.j0 + self.n_local]
        if self.kind != "sparse_sign":
            raise DimensionMismatch("as_sparse only applies to sparse_sign sketches")
        rows = self.n_local
        csr = sp.csr_matrix((self.vals.cpu().numpy().ravel().copy(),
                             self.cols.cpu().numpy().ravel().astype(np.int64),
                             np.arange(0, rows * self.s + 1, self.s)), shape=(rows, self.w))
        csr.sort_indices()
        return csr

    def matvec(self, u: torch.Tensor) -> torch.Tensor:
        """W u for a length-w device vector (local rows)."""
        if u.shape != (self.w,):
            raise DimensionMismatch(f"u has shape {tuple(u.shape)}, expected ({self.w},)")
        if self.kind == "identity":
            return u[self.j0:self.j0 + self.n_local].clone()
        out = torch.empty(self.n_local, dtype=F64, device=u.device)
        if self.kind == "gaussian":  # dense @ u, one warp per row (sketching.py:78-79)
            _lib.call("skb_rowdot_gemv", self.dense, self.w, self.n_local, self.w, 0, u, out,
                      None, stream_ptr())
            return out
        _lib.call("skb_sketch_gather", self.cols, self.vals, self.s, self.n_local, u, None, None,
                  out, stream_ptr())
        return out

    @property
    def n_local(self) -> int:
        if self.cols is not None:
            return int(self.cols.shape[0])
        if self.dense is not None:
            return int(self.dense.shape[0])
        return self.n if self.kind != "identity" else self._n_local

    _n_local: int = 0


def auto_sketch_dims(m: int, n: int, delta: float):
    """Reference auto_sketch_dims (sketching.py:83-90)."""
    lg = max(1, math.ceil(math.log2(m / delta)))
    w = min(n, 8 * m * lg)
    return w, min(max(2, lg), w)


def build_sparse_embedding(n: int, w: int, s: int, seed: int, rows=None,
                           device=None) -> SketchOperator:
    """Sparse sign embedding (sketching.py:93-119) drawn on the GPU.

    rows = (j0, j1) keeps only this rank's rows (the full stream is drawn)."""
    if not (1 <= s <= w):
        raise InvalidDims(f"need 1 <= s <= w, got s={s}, w={w}")
    if w > n * s:
        raise InvalidDims(f"w={w} exceeds n*s={n * s}")
    device = device or require_cuda()
    k0, k1 = philox_key(seed)
    cols, vals, used = K.sparse_embedding(k0, k1, n, w, s, device)
    j0 = 0
    if rows is not None and (rows[0] != 0 or rows[1] != n):
        j0 = rows[0]
        cols = cols[rows[0]:rows[1]].contiguous()
        vals = vals[rows[0]:rows[1]].contiguous()
    return SketchOperator(kind="sparse_sign", n=n, w=w, s=s, seed=int(seed), cols=cols, vals=vals,
                          j0=j0, words_used=used)


def build_identity_sketch(n: int, rows=None) -> SketchOperator:
    """W = I for w >= n (sketching.py:122-128)."""
    if n < 1:
        raise InvalidDims(f"n must be positive, got {n}")
    W = SketchOperator(kind="identity", n=n, w=n, s=0, seed=0)
    W.j0 = rows[0] if rows else 0
    W._n_local = (rows[1] - rows[0]) if rows else n
    return W


ZIG_TILE = 4096            # stream positions per generator tile (csrc/skb_gauss.cu)
ZIG_WORDS_PER_DRAW = 1.03  # stream words per standard_normal draw, with margin (numpy: 1.0220)


def build_gaussian_sketch(n: int, w: int, seed: int, rows=None, device=None,
                          comm=None) -> SketchOperator:
    """Dense Gaussian sketch (sketching.py:131-139): standard_normal((n, w)) / sqrt(w)
    drawn on the GPU bit-exact with numpy's ziggurat (K9, csrc/skb_gauss.cu).
    rows = (j0, j1) keeps this rank's row block (draws j0*w .. j1*w). With an
    active comm every rank generates one slice of the STREAM (not of the draws:
    draw k's stream position depends on all earlier slow attempts), the per-rank
    draw counts give each slice's global draw offset, and one all-to-all moves
    the few draws that landed on a neighbour — no rank walks the whole prefix."""
    if w < 1:
        raise InvalidDims(f"w must be positive, got {w}")
    device = device or require_cuda()
    j0, j1 = rows if rows is not None else (0, n)
    k0, k1 = philox_key(seed)
    if comm is not None and comm.active:
        dense = _gaussian_rows_distributed(k0, k1, n, w, j0, j1, comm, device)
    else:
        dense = torch.empty((j1 - j0, w), dtype=F64, device=device)
        need = _gaussian_ws_bytes(j1 * w, device)
        ws, cap = workspace(need)
        _lib.call("skb_gaussian_sketch", k0, k1, j0 * w, j1 * w, w, dense, ws, cap, stream_ptr())
    return SketchOperator(kind="gaussian", n=n, w=w, s=0, seed=int(seed), dense=dense, j0=j0)


def _gaussian_ws_bytes(count: int, device) -> int:
    """Generator workspace, with the stored-values scratch (8 B per stream
    position; one Philox pass instead of two) when device memory allows it."""
    base = int(_lib.lib().skb_gaussian_workspace_bytes(count))
    extra = int(_lib.lib().skb_gaussian_value_bytes(count))
    free, _ = torch.cuda.mem_get_info(device)
    return base + extra if free > base + extra + (4 << 30) else base


def _gaussian_rows_distributed(k0, k1, n, w, j0, j1, comm, device):
    from .distributed import shard_range
    total = n * w
    ratio = ZIG_WORDS_PER_DRAW
    for _ in range(4):
        ptot = -(-int(total * ratio + 8 * ZIG_TILE) // ZIG_TILE) * ZIG_TILE
        # this rank's stream slice, proportional to its row block
        p0 = (ptot * j0 // n) // ZIG_TILE * ZIG_TILE
        p1 = ptot if j1 == n else (ptot * j1 // n) // ZIG_TILE * ZIG_TILE
        cap = max(1, p1 - p0)  # at most one draw per word
        buf = torch.empty(cap, dtype=F64, device=device)
        need = _gaussian_ws_bytes(cap, device)
        ws, wcap = workspace(need)
        cnt = np.zeros(1, dtype=np.uint64)
        _lib.call("skb_gaussian_range", k0, k1, p0, p1, w, buf, cap, cnt.ctypes.data, ws, wcap,
                  stream_ptr())
        counts = comm.allgather_rows(torch.tensor([int(cnt[0])], dtype=torch.int64,
                                                  device=device), comm.world)
        counts = [int(c) for c in counts.cpu()]
        if sum(counts) >= total:
            break
        ratio *= 1.01  # too few draws in the stream slices: widen and redo (never observed)
    else:
        raise RuntimeError("Gaussian sketch: stream slices never covered n * w draws")
    offs = np.concatenate([[0], np.cumsum(counts)])
    mine0, mine1 = int(offs[comm.rank]), int(offs[comm.rank + 1])  # draws this rank holds
    send, recv = [], []
    for h in range(comm.world):
        a0, a1 = shard_range(n, h, comm.world)
        lo, hi = max(mine0, a0 * w), min(mine1, a1 * w)        # my draws rank h needs
        send.append(max(0, hi - lo))
        lo2, hi2 = max(int(offs[h]), j0 * w), min(int(offs[h + 1]), j1 * w)  # h's draws I need
        recv.append(max(0, hi2 - lo2))
    a_first = max(mine0, shard_range(n, 0, comm.world)[0] * w)
    s0 = a_first - mine0
    out = comm.all_to_all_v(buf[s0:s0 + sum(send)].contiguous(), send, recv)
    return out.reshape(j1 - j0, w)


def apply_sketch(lp, d: torch.Tensor, W: SketchOperator, check_positive: bool = True):
    """X = (A diag(d) W)' as a DeviceMatrix with w 'columns' of length m
    (sketching.py:142-161). lp: DeviceLP (this rank's columns)."""
    A = lp.A
    if d.shape != (A.n,):
        raise DimensionMismatch(f"d has shape {tuple(d.shape)}, expected ({A.n},)")
    if W.n != lp.n:
        raise DimensionMismatch(f"sketch has {W.n} rows, expected {lp.n}")
    if check_positive and lp.vec_stats(d)[3] <= 0.0:
        raise NonpositiveScaling("column scaling d must be strictly positive")
    m = A.m
    ldx = lda_for(m)
    X = torch.empty((W.w, ldx), dtype=F64, device=d.device)
    if W.kind == "identity":  # ADW = AD: X's rows are the scaled columns (w = n)
        if lp.comm.active:
            X.zero_()
        sub = X[lp.j0:lp.j0 + A.n] if lp.comm.active else X
        if lp.sparse:  # scatter the CSC columns straight into X (A is never densified)
            if not lp.comm.active:
                X.zero_()
            _lib.call("skb_csc_to_dense", A.colptr, A.rowidx, A.vals, A.n, sub, ldx, stream_ptr())
            sub[:, :m] *= d[:, None]  # X[j, i] = A_ij * d_j, one rounding as in skb_scale_columns
        else:
            _lib.call("skb_scale_columns", A.cols, m, A.n, A.lda, d, sub, ldx, stream_ptr())
    elif W.kind == "sparse_sign":
        need = int(_lib.lib().skb_sketch_workspace_bytes(A.n, W.w, W.s))
        ws, cap = workspace(need)
        if lp.sparse:  # CSC A (config c4)
            _lib.call("skb_csc_sketch_apply", A.colptr, A.rowidx, A.vals, A.ell(), A.m, A.n, d,
                      W.cols, W.vals, W.s, W.w, X, ldx, ws,
                      cap, stream_ptr())
        else:
            _lib.call("skb_sketch_apply", A.cols, m, A.n, A.lda, d, W.cols, W.vals, W.s, W.w, X,
                      ldx, ws, cap, stream_ptr())
    else:  # dense Gaussian: one DMMA GEMM, X = W' D A' (sketching.py:158-159)
        Ad = lp.dense_A()
        # + room for up to 8 split-K partials of the w x m product, or for the
        # INT8 emulation's residues in K chunks of 65536 (csrc/skb_ozaki.cu)
        L = _lib.lib()
        need = max(8 * 8 * m * W.w, int(L.skb_gemm_ozaki_workspace_bytes(W.w, m, min(Ad.n, 65536))))
        ws, cap = workspace(int(L.skb_factor_workspace_bytes(m, W.w)) + need)
        _lib.call("skb_gaussian_apply", Ad.cols, m, Ad.n, Ad.lda, d, W.dense, W.w, X, ldx, ws,
                  cap, stream_ptr())
    if ldx != m:
        X[:, m:].zero_()
    if lp.comm.active:
        if W.kind == "identity" or not DISTRIBUTED_FACTOR:
            lp.comm.allreduce_(X)
        else:
            # ADW = sum_g A_g D_g W_g: reduce-scatter by bucket (row) blocks; the
            # factor is then built from the blocks (preconditioning.py)
            r0, _ = lp.comm.row_block(W.w)
            Xd = K.DeviceMatrix(lp.comm.reduce_scatter_rows(X), m)
            Xd.dist = (W.w, r0, lp.comm)
            return Xd
    return K.DeviceMatrix(X, m)
