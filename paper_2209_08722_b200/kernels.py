"""Thin typed wrappers over the libskb C ABI (device tensors in, device tensors out).

Each wrapper names the reference call it replaces. Higher layers
(sketching, krylov_solvers, ipm_core) only talk to the device through here.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .runtime import F64, lda_for, require_cuda, stream_ptr, workspace


class DeviceMatrix:
    """Dense A (m x n) stored column-major on the device.

    `cols` is a (n, lda) float64 tensor whose row j is column j of A (zero
    padded to lda = m rounded up to even). Column blocks are contiguous so the
    streaming kernels move them with the TMA bulk engine."""

    def __init__(self, cols: torch.Tensor, m: int):
        assert cols.dtype == F64 and cols.is_cuda and cols.dim() == 2
        assert cols.shape[1] == lda_for(m) and cols.is_contiguous()
        self.cols = cols
        self.m = int(m)
        self.n = int(cols.shape[0])
        self.lda = int(cols.shape[1])

    @property
    def shape(self):
        return (self.m, self.n)

    @classmethod
    def from_host(cls, A, device=None) -> "DeviceMatrix":
        """A: numpy (m x n) dense, or a scipy sparse matrix (densified)."""
        device = device or require_cuda()
        if hasattr(A, "toarray"):
            A = A.toarray()
        A = np.asarray(A, dtype=np.float64)
        m, n = A.shape
        if A.flags.c_contiguous and 8 * m * n >= (1 << 30):
            free, _ = torch.cuda.mem_get_info(device)
            if free > 2.2 * 8 * m * n:  # row-major upload, transpose in HBM
                rows = torch.empty((m, n), dtype=F64, device=device)
                step = max(1, (1 << 28) // (8 * n))
                for i0 in range(0, m, step):
                    rows[i0:i0 + step].copy_(torch.from_numpy(A[i0:i0 + step]))
                out = cls.from_rows_device(rows)
                del rows
                return out
        cols = torch.zeros((n, lda_for(m)), dtype=F64, device=device)
        step = max(1, (1 << 28) // max(1, 8 * m))  # upload in ~256 MB column slabs
        for j0 in range(0, n, step):
            j1 = min(n, j0 + step)
            blk = torch.from_numpy(np.ascontiguousarray(A[:, j0:j1].T))
            cols[j0:j1, :m].copy_(blk, non_blocking=False)
        return cls(cols, m)

    @classmethod
    def from_rows_device(cls, A_rows: torch.Tensor) -> "DeviceMatrix":
        """A given as a (m x n) row-major device tensor."""
        m, n = A_rows.shape
        cols = torch.zeros((n, lda_for(m)), dtype=F64, device=A_rows.device)
        cols[:, :m].copy_(A_rows.t())
        return cls(cols, m)

    def column_slice(self, j0: int, j1: int) -> "DeviceMatrix":
        return DeviceMatrix(self.cols[j0:j1], self.m)

    def to_host(self) -> np.ndarray:
        return self.cols[:, : self.m].t().contiguous().cpu().numpy()


def _ws(m: int, extra: int = 0):
    need = int(_lib.lib().skb_stream_workspace_bytes(m)) + extra
    return workspace(need)


def _p(t):
    return None if t is None else t


class SparseDeviceMatrix:
    """Sparse A (m x n) stored as CSC on the device (config c4): colptr int64
    (n+1), rowidx int32, vals float64. Column slices share the arrays."""

    is_sparse = True

    def __init__(self, colptr: torch.Tensor, rowidx: torch.Tensor, vals: torch.Tensor, m: int):
        self.colptr, self.rowidx, self.vals = colptr, rowidx, vals
        self.m = int(m)
        self.n = int(colptr.numel() - 1)
        self.lda = None

    @property
    def shape(self):
        return (self.m, self.n)

    @classmethod
    def from_host(cls, A, device=None) -> "SparseDeviceMatrix":
        import scipy.sparse as sp
        device = device or require_cuda()
        csc = sp.csc_matrix(A, dtype=np.float64)
        csc.sort_indices()
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)  # noqa
        return cls(t(csc.indptr, np.int64), t(csc.indices, np.int32), t(csc.data, np.float64),
                   csc.shape[0])

    def args(self):
        return (self.colptr, self.rowidx, self.vals, self.m, self.n)

    def pargs(self):
        """args() with the pass plan of the deterministic (atomic-free) CSC
        passes (csrc/skb_cscplan.cuh) when one was built, else (None, 0): the
        thread-per-column passes with shared-memory atomics."""
        plan, nch = getattr(self, "_plan", None) or self.plan()
        return (self.colptr, self.rowidx, self.vals, plan, nch, self.ell(), self.m, self.n)

    def ell(self):
        """ELL head records (skb_csc_ell_build, one 64-byte record per column),
        built once per matrix; None where they do not apply (m > 65535) or when
        SKB_CSC_ELL=0."""
        if not hasattr(self, "_ell"):
            import os
            self._ell = None
            nb = int(_lib.lib().skb_csc_ell_bytes(self.m, self.n)) if self.n > 0 else 0
            if nb > 0 and os.environ.get("SKB_CSC_ELL", "1") != "0":
                buf = torch.empty(nb, dtype=torch.uint8, device=self.vals.device)
                _lib.call("skb_csc_ell_build", self.colptr, self.rowidx, self.vals, self.m,
                          self.n, buf, nb, stream_ptr())
                self._ell = buf
        return self._ell

    DET_MAX_NNZ = 1 << 24

    def plan(self, force: bool = False):
        """Build (once) the pass plan of the deterministic CSC passes. Default:
        for matrices up to DET_MAX_NNZ nonzeros, whose passes are launch-bound
        anyway, so every CSC result there is bitwise reproducible run to run;
        above it (c4: 1e8 nnz) the shared-atomic passes, which are faster
        (0.47 vs 0.69 ms at c4) but sum in arbitration order.
        SKB_CSC_PLAN=1 plans every matrix, SKB_CSC_PLAN=0 none."""
        import os
        env = os.environ.get("SKB_CSC_PLAN", "")
        if getattr(self, "_plan", None) is None or (
                (force or env == "1") and self._plan[0] is None
                and not getattr(self, "_plan_tried", False)):
            self._plan = (None, 0)
            nnz = int((self.colptr[-1] - self.colptr[0]).item()) if self.n > 0 else 0
            want = force or env == "1" or (env != "0" and nnz <= self.DET_MAX_NNZ)
            if want and self.n > 0:
                self._plan_tried = True
                lens = self.colptr[1:] - self.colptr[:-1]
                maxlen = int(lens.max().item())
                nb = int(_lib.lib().skb_csc_plan_bytes(self.m, self.n, nnz, maxlen))
                if nb > 0:
                    buf = torch.empty(nb, dtype=torch.uint8, device=self.vals.device)
                    nch = np.zeros(1, dtype=np.int64)
                    _lib.call("skb_csc_plan_build", self.colptr, self.rowidx, self.vals, self.m,
                              self.n, nnz, maxlen, buf, nb, nch.ctypes.data, stream_ptr())
                    self._plan = (buf, int(nch[0]))
        return self._plan

    def to_host(self):
        """scipy CSC copy (column slices rebased to their first entry)."""
        import scipy.sparse as sp
        ptr = self.colptr.cpu().numpy()
        a, b = int(ptr[0]), int(ptr[-1])
        return sp.csc_matrix((self.vals[a:b].cpu().numpy(), self.rowidx[a:b].cpu().numpy(),
                              ptr - a), shape=(self.m, self.n))

    def to_dense(self) -> "DeviceMatrix":
        """Dense column-major copy on the device (for the dense-only paths)."""
        cols = torch.zeros((self.n, lda_for(self.m)), dtype=F64, device=self.vals.device)
        _lib.call("skb_csc_to_dense", self.colptr, self.rowidx, self.vals, self.n, cols,
                  cols.shape[1], stream_ptr())
        return DeviceMatrix(cols, self.m)


def _amat(A, planned: bool = True):
    """-> (C symbol prefix, leading C arguments) for a dense or CSC matrix
    (CSC passes that produce an m-vector take the matrix's pass plan)."""
    if getattr(A, "is_sparse", False):
        return "skb_csc_", (A.pargs() if planned else A.args())
    return "skb_", (A.cols, A.m, A.n, A.lda)


def normal_apply(A, d2, z, out, sub=None, gate=None):
    """out = A (d2 .* (A' z)) [- sub]   (krylov_solvers.py:46-47)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "normal_apply", *args, d2, z, out, _p(sub), gate, ws, cap, stream_ptr())
    return out


def gemv(A, x, out, sub=None):
    """out = A x [- sub]   (lp.A @ x, ipm_core.py:99)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "gemv", *args, x, out, _p(sub), ws, cap, stream_ptr())
    return out


def gemv_ratio(A, v, s, out, sub=None):
    """out = A (v / s) [- sub]   (ipm_core.py:502)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "gemv_ratio", *args, v, s, out, _p(sub), ws, cap, stream_ptr())
    return out


def rhs(A, x, s, sigma_mu: float, out, r_d=None, r_p=None):
    """build_rhs (ipm_core.py:196-206)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "rhs", *args, x, s, _p(r_d), float(sigma_mu), out, _p(r_p), ws, cap,
              stream_ptr())
    return out


def gemv_t(A, y, out, add=None, sub=None):
    """out = (A' y [+ add]) [- sub]   (ipm_core.py:100,218)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "gemv_t", *args, y, _p(add), _p(sub), out, ws, cap, stream_ptr())
    return out


def directions(A, dy, x, s, v, sigma_mu, ds, dx, adx, atdy=None, r_d=None):
    """assemble_directions' A-passes in one sweep (ipm_core.py:218-223)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "directions", *args, dy, x, s, v, _p(r_d), float(sigma_mu), ds, dx, _p(atdy),
              adx, ws, cap, stream_ptr())


def directions_v(A, dy, x, s, v, sigma_mu, ds, dx, adx, avs, atdy=None, r_d=None) -> bool:
    """directions() plus avs = A (v / s) in the same pass (ipm_core.py:218-223, :502);
    False where the fused pass does not apply (CSC, m > 2048): use the two passes."""
    if isinstance(A, SparseDeviceMatrix) or A.m > 2048:
        return False
    ws, cap = _ws(A.m)
    try:
        _lib.call("skb_directions_v", A.cols, A.m, A.n, A.lda, dy, x, s, v, _p(r_d),
                  float(sigma_mu), ds, dx, _p(atdy), adx, avs, ws, cap, stream_ptr())
    except _lib.SkbError as e:
        if e.code == -6:  # SKB_ERR_UNSUPPORTED: the caller runs the two passes
            return False
        raise
    return True


def iterate_rhs(A, xn, sn, y_new, c, smu_dev, infeasible: bool, r_p, r_d, p, b=None,
                p_sub_rp: bool = False) -> bool:
    """make_iterate's pass at (xn, sn) fused with the next step's build_rhs
    (skb_iterate_rhs); False where it does not apply (CSC, m > 2048)."""
    if isinstance(A, SparseDeviceMatrix) or A.m > 2048:
        return False
    ws, cap = _ws(A.m)
    try:
        _lib.call("skb_iterate_rhs", A.cols, A.m, A.n, A.lda, xn, sn, y_new, c, smu_dev,
                  1 if infeasible else 0, _p(b), r_p, r_d, p, 1 if p_sub_rp else 0, ws, cap,
                  stream_ptr())
    except _lib.SkbError as e:
        if e.code == -6:  # SKB_ERR_UNSUPPORTED
            return False
        raise
    return True


def iterate(A, x, s, y_new, b, c, r_p, r_d, dx=None, ds=None, alpha=0.0, x_out=None,
            s_out=None):
    """make_iterate's A-passes in one sweep (ipm_core.py:94-102)."""
    ws, cap = _ws(A.m)
    pre, args = _amat(A)
    _lib.call(pre + "iterate", *args, x, _p(dx), s, _p(ds), float(alpha), y_new, b, c,
              _p(x_out), _p(s_out), r_p, r_d, ws, cap, stream_ptr())


def sparse_embedding(key0: int, key1: int, n: int, w: int, s: int, device=None):
    """build_sparse_embedding's draws (sketching.py:104-117) -> (cols int32 (n,s), vals f64 (n,s), words)."""
    device = device or require_cuda()
    cols = torch.empty((n, s), dtype=torch.int32, device=device)
    vals = torch.empty((n, s), dtype=F64, device=device)
    ws_need = 64 * n * max(s, 1) + (1 << 20)
    ws, cap = workspace(ws_need)
    used = np.zeros(1, dtype=np.uint64)
    _lib.call("skb_sparse_embedding", key0, key1, n, w, s, cols, vals, used.ctypes.data, ws, cap,
              stream_ptr())
    return cols, vals, int(used[0])


def lemire_draw(key0: int, key1: int, bound: int, count: int, word_offset: int = 0,
                device=None):
    """rng.integers(0, bound, count) from 32-bit word `word_offset` -> (uint32 as int64, words)."""
    device = device or require_cuda()
    out = torch.empty(count, dtype=torch.int32, device=device)
    ws, cap = workspace(64 * count + (1 << 20))
    used = np.zeros(1, dtype=np.uint64)
    _lib.call("skb_lemire_draw", key0, key1, word_offset, bound, count, out, used.ctypes.data, ws,
              cap, stream_ptr())
    return out.to(torch.int64) & 0xFFFFFFFF, int(used[0])
