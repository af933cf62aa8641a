"""Seeded synthetic LP generators for the BASELINE configurations (host side).

Harness code shared by the parity tests, the oracle and bench.py. Draw order
follows SURVEY.md §8(d) so the host bits are identical on every side:

    G = Generator(Philox(seed))
    A  = G.standard_normal((m, n))            (dense configs c1/c2/c3)
    y0 = G.standard_normal(m); x0 = G.uniform(0.5, 1.5, n); s0 = G.uniform(0.5, 1.5, n)
    b  = A @ x0;  c = A.T @ y0 + s0

The configurations quote gamma = 0.1, but their start has theta0 =
min(x0*s0)/mu0 ~ 0.26, so the reference's feasible mode rejects it
(ipm_core.py:688-689). Following the reference's own widening rule
(ipm_core.py:693-698) the run uses gamma_run = max(gamma, 1 - 0.999*theta0)
(SURVEY.md Appendix C).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class DenseLP:
    """min c'x s.t. Ax = b, x >= 0 with dense row-major A (m x n) and a
    strictly feasible start (x0, y0, s0)."""

    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    x0: np.ndarray
    y0: np.ndarray
    s0: np.ndarray
    name: str = "dense_lp"

    @property
    def m(self) -> int:
        return self.A.shape[0]

    @property
    def n(self) -> int:
        return self.A.shape[1]

    def theta0(self) -> float:
        xs = self.x0 * self.s0
        return float(np.min(xs) / (float(self.x0 @ self.s0) / self.n))

    def gamma_run(self, gamma: float) -> float:
        return max(gamma, 1.0 - 0.999 * self.theta0())


def wide_dense_lp(m: int, n: int, seed: int = 0) -> DenseLP:
    """configs c1/c2/c3 (BASELINE.json): A iid N(0,1), feasible start."""
    g = np.random.Generator(np.random.Philox(int(seed)))
    A = g.standard_normal((m, n))
    y0 = g.standard_normal(m)
    x0 = g.uniform(0.5, 1.5, n)
    s0 = g.uniform(0.5, 1.5, n)
    b = A @ x0
    c = A.T @ y0 + s0
    return DenseLP(A, b, c, x0, y0, s0, name=f"wide_dense_{m}x{n}_s{seed}")


@dataclass
class SparseLP:
    """Config c4: A (m x n, scipy CSC) with k nonzeros per column, feasible start."""

    A: object
    b: np.ndarray
    c: np.ndarray
    x0: np.ndarray
    y0: np.ndarray
    s0: np.ndarray
    name: str = "sparse_lp"

    @property
    def m(self) -> int:
        return self.A.shape[0]

    @property
    def n(self) -> int:
        return self.A.shape[1]

    def theta0(self) -> float:
        return float(np.min(self.x0 * self.s0) / (float(self.x0 @ self.s0) / self.n))

    def gamma_run(self, gamma: float) -> float:
        return max(gamma, 1.0 - 0.999 * self.theta0())


def sparse_wide_lp(m: int, n: int, k: int = 5, seed: int = 0) -> SparseLP:
    """config c4: per column k distinct rows from
    G.integers(0, m, (n, k)) with duplicate rows redrawn, values
    G.standard_normal((n, k)), then y0, x0, s0 as for the dense configs."""
    import scipy.sparse as sp
    g = np.random.Generator(np.random.Philox(int(seed)))
    rows = g.integers(0, m, size=(n, k))
    while True:
        dup = (np.diff(np.sort(rows, axis=1), axis=1) == 0).any(axis=1)
        if not dup.any():
            break
        rows[dup] = g.integers(0, m, size=(int(dup.sum()), k))
    vals = g.standard_normal((n, k))
    y0 = g.standard_normal(m)
    x0 = g.uniform(0.5, 1.5, n)
    s0 = g.uniform(0.5, 1.5, n)
    colptr = np.arange(0, n * k + 1, k, dtype=np.int64)
    A = sp.csc_matrix((vals.ravel(), rows.ravel(), colptr), shape=(m, n))
    A.sort_indices()
    b = A @ x0
    c = A.T @ y0 + s0
    return SparseLP(A, b, c, x0, y0, s0, name=f"sparse_wide_{m}x{n}_k{k}_s{seed}")


def random_feasible_dense(m: int, n: int, density: float, seed: int):
    """The reference's random_feasible_lp instance (lp_model.py:134-160), same
    draw order: mask, values, diagonal boost, x_feas, y0, slack. Returns dense
    (A, b, c); used by the feasible-start parity tests (no start supplied)."""
    g = np.random.Generator(np.random.Philox(int(seed)))
    keep = g.random((m, n)) < density
    A = np.where(keep, g.random((m, n)), 0.0)
    k = min(m, n)
    A[np.arange(k), np.arange(k)] += g.random(k)
    x_feas = g.random(n) + 0.5
    b = A @ x_feas
    y0 = g.standard_normal(m)
    c = A.T @ y0 + g.random(n) + 0.1
    return A, b, c


def random_dense(m: int, n: int, density: float, seed: int):
    """The reference's random_lp instance (lp_model.py:113-135): same draw
    order (mask, values, diagonal boost, x0, z, c); b = A x0 + 0.1 z is
    sign-indefinite against A >= 0, so such draws are infeasible almost surely.
    Returns dense (A, b, c)."""
    g = np.random.Generator(np.random.Philox(int(seed)))
    keep = g.random((m, n)) < density
    A = np.where(keep, g.random((m, n)), 0.0)
    k = min(m, n)
    A[np.arange(k), np.arange(k)] += g.random(k)
    x0 = g.standard_normal(n)
    z = g.standard_normal(m)
    b = A @ x0 + 0.1 * z
    c = g.standard_normal(n)
    return A, b, c


def ill_conditioned_lp(m: int, n: int, seed: int = 0) -> DenseLP:
    """config c5 with the repaired start of SURVEY.md Appendix C:
    A = diag(r) G, r log-uniform on [1e-3, 1e3]; x0, s0 ~ U(0.5, 1.5)."""
    g = np.random.Generator(np.random.Philox(int(seed)))
    G = g.standard_normal((m, n))
    r = 10.0 ** g.uniform(-3.0, 3.0, m)
    A = r[:, None] * G
    y0 = g.standard_normal(m)
    x0 = g.uniform(0.5, 1.5, n)
    s0 = g.uniform(0.5, 1.5, n)
    b = A @ x0
    c = A.T @ y0 + s0
    return DenseLP(A, b, c, x0, y0, s0, name=f"ill_cond_{m}x{n}_s{seed}")
