"""LP containers: the reference's host-side LinearProgram and its device mirror.

`LinearProgram`, `make_lp` and `validate` keep the reference's API
(reference lp_model.py:34-49,76-106) so callers can hand the same object to
either implementation. `DeviceLP` is the B200 layout the hot path runs on:
A column-major in HBM (a column-sharded block per rank), b replicated, c and
every n-vector sharded like A's columns. All comm-aware A-passes live here:
an m-vector output is a local column-block sum, allreduced across ranks,
then `sub` is subtracted.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from . import kernels as K
from .distributed import MAX, MIN, SUM, Comm
from .errors import DimensionMismatch, ZeroRow
from .runtime import F64, require_cuda, stream_ptr, to_host, workspace


SPARSE_DENSITY = 0.1  # CSC device storage below this fill (12 B/nnz vs 8 B/entry dense)


@dataclass
class LinearProgram:
    """min c'x s.t. Ax = b, x >= 0; A is scipy CSR or a dense numpy array."""

    A: object
    b: np.ndarray
    c: np.ndarray
    name: str = "lp"

    @property
    def m(self) -> int:
        return self.A.shape[0]

    @property
    def n(self) -> int:
        return self.A.shape[1]


def make_lp(A, b, c, name: str = "lp") -> LinearProgram:
    """Reference make_lp (lp_model.py:76-83): CSR storage, validated."""
    A = sp.csr_matrix(A, dtype=np.float64)
    A.sort_indices()
    lp = LinearProgram(A, np.asarray(b, dtype=np.float64), np.asarray(c, dtype=np.float64), name)
    validate(lp)
    return lp


def validate(lp: LinearProgram) -> None:
    """Reference validate (lp_model.py:86-106): shapes, n >= m, finiteness, no zero rows."""
    m, n = lp.A.shape
    if m < 1:
        raise DimensionMismatch("m must be at least 1")
    if n < m:
        raise DimensionMismatch(f"wide problem required: n={n} < m={m}")
    if np.shape(lp.b) != (m,):
        raise DimensionMismatch(f"b has shape {np.shape(lp.b)}, expected ({m},)")
    if np.shape(lp.c) != (n,):
        raise DimensionMismatch(f"c has shape {np.shape(lp.c)}, expected ({n},)")
    data = lp.A.data if sp.issparse(lp.A) else np.asarray(lp.A)
    if not (np.all(np.isfinite(lp.b)) and np.all(np.isfinite(lp.c)) and np.all(np.isfinite(data))):
        raise ValueError("problem data contains nonfinite entries")
    if sp.issparse(lp.A):
        rmax = abs(lp.A).max(axis=1).toarray().ravel()
    else:
        rmax = np.abs(np.asarray(lp.A)).max(axis=1)
    zero = np.where(rmax == 0.0)[0]
    if zero.size:
        raise ZeroRow(int(zero[0]))


def random_lp(m: int, n: int, density: float, seed: int) -> LinearProgram:
    """Reference random_lp (lp_model.py:113-135): same generator and draw order
    (problems.random_dense); sign-indefinite b, so infeasible almost surely."""
    from .errors import InvalidDensity
    from .problems import random_dense
    if not 0.0 < density <= 1.0:
        raise InvalidDensity(f"density {density} outside (0, 1]")
    if n < m:
        raise DimensionMismatch(f"wide problem required: n={n} < m={m}")
    A, b, c = random_dense(m, n, density, seed)
    return make_lp(A, b, c, name=f"random_lp_{m}x{n}_d{density}_s{seed}")


def random_feasible_lp(m: int, n: int, density: float, seed: int) -> LinearProgram:
    """Reference random_feasible_lp (lp_model.py:138-160): strictly feasible primal
    and dual by construction (problems.random_feasible_dense)."""
    from .errors import InvalidDensity
    from .problems import random_feasible_dense
    if not 0.0 < density <= 1.0:
        raise InvalidDensity(f"density {density} outside (0, 1]")
    A, b, c = random_feasible_dense(m, n, density, seed)
    return make_lp(A, b, c, name=f"random_feasible_lp_{m}x{n}_d{density}_s{seed}")


def _dev(a, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=F64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)


class DeviceLP:
    """Device-resident LP (this rank's column block)."""

    def __init__(self, A: K.DeviceMatrix, b: torch.Tensor, c_local: torch.Tensor, n: int,
                 j0: int, comm: Comm, name: str = "lp"):
        self.A = A
        self.b = b
        self.c = c_local
        self.m = A.m
        self.n = int(n)
        self.n_local = A.n
        self.j0 = int(j0)
        self.comm = comm
        self.name = name
        self.device = b.device
        # scales used by the reference's checks
        st = self.vec_stats(self.b, global_=False)
        self.b_norm = math.sqrt(st[0])
        self.c_norm = math.sqrt(self.vec_stats(self.c)[0])
        self.sparse = bool(getattr(A, "is_sparse", False))
        self.a_scale = math.sqrt(self.vec_stats(A.vals if self.sparse else A.cols.view(-1))[0])
        self._dense = None

    def dense_A(self) -> "K.DeviceMatrix":
        """A in the dense column-major layout (a device-side copy for CSC inputs,
        used by the dense-only paths: direct solver, phase 1, Gaussian GEMM)."""
        if not self.sparse:
            return self.A
        if self._dense is None:
            self._dense = self.A.to_dense()
        return self._dense

    # ---------------------------------------------------------- construction
    @classmethod
    def from_host(cls, lp, comm: Comm | None = None, device=None) -> "DeviceLP":
        """lp: LinearProgram (CSR or dense A) or any object with A, b, c."""
        comm = comm or Comm()
        device = device or require_cuda()
        A = lp.A
        m, n = A.shape
        j0, j1 = comm.shard(n)
        if sp.issparse(A):
            blk = A.tocsc()[:, j0:j1]
            # genuinely sparse inputs stay CSC on the device (config c4); dense data that
            # arrives as CSR (make_lp always stores CSR) is streamed column-major
            density = blk.nnz / max(1, blk.shape[0] * blk.shape[1])
            Ad = (K.SparseDeviceMatrix.from_host(blk, device) if density < SPARSE_DENSITY
                  else K.DeviceMatrix.from_host(blk, device))
        else:
            Ad = K.DeviceMatrix.from_host(np.asarray(A)[:, j0:j1], device)
        return cls(Ad, _dev(lp.b, device), _dev(np.asarray(lp.c)[j0:j1], device), n, j0, comm,
                   getattr(lp, "name", "lp"))

    @classmethod
    def from_device(cls, A: K.DeviceMatrix, b, c_local, n: int, j0: int = 0,
                    comm: Comm | None = None, name="lp") -> "DeviceLP":
        return cls(A, b, c_local, n, j0, comm or Comm(), name)

    def local(self, v) -> torch.Tensor:
        """Slice a full-length host/device n-vector to this rank's columns."""
        if isinstance(v, torch.Tensor) and v.numel() == self.n_local and v.is_cuda:
            return v.to(F64).contiguous()
        arr = v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v)
        if arr.shape[0] == self.n:
            arr = arr[self.j0:self.j0 + self.n_local]
        return _dev(arr, self.device)

    def new_n(self):
        return torch.empty(self.n_local, dtype=F64, device=self.device)

    def new_m(self):
        return torch.empty(self.m, dtype=F64, device=self.device)

    # -------------------------------------------------- comm-aware A-passes
    def _finish_m(self, out, sub):
        if self.comm.active:
            self.comm.allreduce_(out)
            if sub is not None:
                _lib.call("skb_sub", out, sub, out, self.m, stream_ptr())
        return out

    def _sub_arg(self, sub):
        return None if self.comm.active else sub

    def gemv(self, x, out=None, sub=None):
        out = self.new_m() if out is None else out
        K.gemv(self.A, x, out, sub=self._sub_arg(sub))
        return self._finish_m(out, sub)

    def gemv_ratio(self, v, s, out=None, sub=None):
        out = self.new_m() if out is None else out
        K.gemv_ratio(self.A, v, s, out, sub=self._sub_arg(sub))
        return self._finish_m(out, sub)

    def normal(self, d2, z, out=None, sub=None, gate=None):
        out = self.new_m() if out is None else out
        K.normal_apply(self.A, d2, z, out, sub=self._sub_arg(sub), gate=gate)
        return self._finish_m(out, sub)

    def rhs(self, x, s, sigma_mu, r_d=None, r_p=None, out=None):
        out = self.new_m() if out is None else out
        K.rhs(self.A, x, s, sigma_mu, out, r_d=r_d, r_p=self._sub_arg(r_p))
        return self._finish_m(out, r_p)

    def gemv_t(self, y, out=None, add=None, sub=None):
        out = self.new_n() if out is None else out
        return K.gemv_t(self.A, y, out, add=add, sub=sub)

    def directions(self, dy, x, s, v, sigma_mu, r_d=None):
        ds, dx, atdy, adx = self.new_n(), self.new_n(), self.new_n(), self.new_m()
        K.directions(self.A, dy, x, s, v, sigma_mu, ds, dx, adx, atdy=atdy, r_d=r_d)
        self._finish_m(adx, None)
        return dx, ds, atdy, adx

    def directions_v(self, dy, x, s, v, sigma_mu, r_d=None, sub=None):
        """directions() and A (v / s) [- sub] from one pass over A, or None where
        the fused pass does not apply (then: directions() and gemv_ratio())."""
        ds, dx, atdy, adx, avs = self.new_n(), self.new_n(), self.new_n(), self.new_m(), \
            self.new_m()
        if not K.directions_v(self.A, dy, x, s, v, sigma_mu, ds, dx, adx, avs, atdy=atdy,
                              r_d=r_d):
            return None
        self._finish_m(adx, None)
        if self.comm.active:
            self._finish_m(avs, sub)
        elif sub is not None:
            _lib.call("skb_sub", avs, sub, avs, self.m, stream_ptr())
        return (dx, ds, atdy, adx), avs

    def iterate(self, x, s, y_new, dx=None, ds=None, alpha=0.0):
        """-> (x_new, s_new, r_p, r_d) of make_iterate at the step."""
        xo = self.new_n() if dx is not None else x
        so = self.new_n() if ds is not None else s
        r_p, r_d = self.new_m(), self.new_n()
        K.iterate(self.A, x, s, y_new, self._sub_arg(self.b), self.c, r_p, r_d,
                  dx=dx, ds=ds, alpha=alpha, x_out=xo if dx is not None else None,
                  s_out=so if ds is not None else None)
        if self.comm.active:
            self._finish_m(r_p, self.b)
        return xo, so, r_p, r_d

    def iterate_with_rhs(self, x, s, y_new, dx, ds, alpha, sigma, infeasible):
        """iterate() at the step plus the next step's rhs from the same pass over A
        (bitwise iterate() followed by rhs() at the new point, whose sigma * mu is
        formed on the device from the same reduction the host's mu comes from):
        -> (x_new, s_new, r_p, r_d, p) or None where the fused pass does not apply."""
        if self.sparse or self.m > 2048:
            return None
        xo, so = self.new_n(), self.new_n()
        _lib.call("skb_step_xs", x, dx, s, ds, float(alpha), xo, so, xo.numel(), stream_ptr())
        st0 = reduce_call("skb_iter_stats", 5, xo, so, None, xo.numel())
        self.comm.combine_(st0, (SUM, MIN, MIN, MIN, SUM))
        smu = torch.empty(1, dtype=F64, device=self.device)
        _lib.call("skb_sigma_mu", st0, float(self.n), float(sigma), smu, stream_ptr())
        r_p, r_d, p = self.new_m(), self.new_n(), self.new_m()
        if not K.iterate_rhs(self.A, xo, so, y_new, self.c, smu, infeasible, r_p, r_d, p,
                             b=self._sub_arg(self.b),
                             p_sub_rp=infeasible and not self.comm.active):
            return None
        if self.comm.active:
            self._finish_m(r_p, self.b)
            self._finish_m(p, r_p if infeasible else None)
        return xo, so, r_p, r_d, p

    # ------------------------------------------------------- reductions
    def vec_stats(self, a, sub=None, global_=True):
        """{sum t^2, sum t, max|t|, min t} of t = a - sub over the global vector."""
        out = reduce_call("skb_vec_stats", 4, a, sub, a.numel())
        if global_:
            self.comm.combine_(out, (SUM, SUM, MAX, MIN))
        return to_host(out)

    def norm_m(self, a, sub=None) -> float:
        """||a - sub|| of a replicated m-vector (no communication)."""
        return math.sqrt(self.vec_stats(a, sub, global_=False)[0])


_RED = threading.local()


def reduction_ws():
    """Per-thread, per-device reduction scratch whose ticket word starts (and
    stays) zero (solves may run from a thread pool, oracle_bench.py:236)."""
    cache = getattr(_RED, "d", None)
    if cache is None:
        cache = _RED.d = {}
    dev = torch.cuda.current_device()
    buf = cache.get(dev)
    if buf is None:
        nb = int(_lib.lib().skb_reduce_workspace_bytes())
        buf = torch.zeros(nb, dtype=torch.uint8, device=require_cuda())
        cache[dev] = buf
    return buf


def reduce_call(fn: str, k: int, *args):
    """Run a libskb reduction kernel; -> device tensor of its k outputs."""
    out = torch.empty(k, dtype=F64, device=require_cuda())
    ws = reduction_ws()
    _lib.call(fn, *args, out, ws, ws.numel(), stream_ptr())
    return out
