"""Planned CSC passes (csrc/skb_cscplan.cuh `cscp_kernel`): the scatter of every
m-vector-producing pass over each chunk's row-sorted products, with fixed
row blocks per scatter warp (no atomics, deterministic). Checked against scipy in
float64 (the reference's NormalOperator.apply, krylov_solvers.py:46-47, and the
A-passes of ipm_core.py:94-102,196-242), against the thread-per-column atomic
kernel, and for bitwise run-to-run determinism, on ragged shapes: empty
columns, long columns, a single row, a single column, long empty runs,
duplicate-free random rows, columns whose length forces the fallback."""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_08722_b200 import kernels
    return kernels


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _h(t):
    return t.detach().cpu().numpy()


def _ragged(m, n, seed, maxlen=40, empty=0.2):
    g = np.random.Generator(np.random.Philox(seed))
    lens = g.integers(0, maxlen + 1, n)
    lens[g.random(n) < empty] = 0
    lens = np.minimum(lens, m)
    if n > 10:
        lens[n // 3: n // 3 + min(5000, n // 4)] = 0  # a long run of empty columns
    rows = [np.sort(g.choice(m, size=int(k), replace=False)) for k in lens]
    colptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ri = np.concatenate(rows).astype(np.int64) if colptr[-1] else np.zeros(0, np.int64)
    return sp.csc_matrix((g.standard_normal(int(colptr[-1])), ri, colptr), shape=(m, n))


CASES = [
    ("c4-like", lambda: _ragged(10_000, 300_000, 1, maxlen=9, empty=0.0)),
    ("ragged", lambda: _ragged(3000, 40_000, 2, maxlen=60)),
    ("long-cols", lambda: _ragged(2500, 3000, 3, maxlen=1000)),
    ("one-row", lambda: _ragged(1, 50_000, 4, maxlen=1)),
    ("one-col", lambda: _ragged(700, 1, 5, maxlen=700, empty=0.0)),
    ("dense-ish", lambda: _ragged(300, 5000, 6, maxlen=300, empty=0.0)),
]


@pytest.mark.parametrize("variant", ["plan", "ell", "plain"])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_planned_passes(K, name, make, variant):
    """variant: plan = the deterministic planned passes (+ ELL records for A'y);
    ell = the atomic passes reading 64-byte ELL records; plain = the atomic
    passes walking colptr -> rowidx -> vals."""
    A = make()
    m, n = A.shape
    g = np.random.Generator(np.random.Philox(8))
    d = 10.0 ** g.uniform(-3, 3, n)
    z, y, b = g.standard_normal(m), g.standard_normal(m), g.standard_normal(m)
    x, s, c = g.random(n) + 0.2, g.random(n) + 0.2, g.standard_normal(n)
    v = 1e-3 * g.standard_normal(n)
    Ad = K.SparseDeviceMatrix.from_host(A)
    if variant == "plan":
        plan, nch = Ad.plan(force=True)
        assert plan is not None and nch > 0, "the plan applies to every case here"
    else:
        Ad._plan, nch = (None, 0), 0
        if variant == "plain":
            Ad._ell = None
        else:
            assert Ad.ell() is not None
    Af = K.SparseDeviceMatrix.from_host(A)
    Af._plan = (None, 0)  # the thread-per-column atomic kernel
    Af._ell = None
    u1 = torch.empty(m, dtype=torch.float64, device="cuda")
    u2 = torch.empty_like(u1)
    # normal operator vs scipy (float64) and vs the atomic kernel
    K.normal_apply(Ad, _t(d * d), _t(z), u1)
    ref = A @ (d * d * (A.T @ z))
    scale = abs(A) @ (d * d * (abs(A.T) @ abs(z))) + 1e-300
    err = np.max(np.abs(_h(u1) - ref) / scale)
    K.normal_apply(Af, _t(d * d), _t(z), u2)
    err2 = np.max(np.abs(_h(u1) - _h(u2)) / scale)
    print(f"{name}/{variant}: m={m} n={n} nnz={A.nnz} chunks={nch} normal err {err:.2e} "
          f"vs atomic {err2:.2e}")
    assert err <= 1e-13 and err2 <= 1e-13
    if variant == "plan":  # bitwise deterministic run to run
        for _ in range(3):
            K.normal_apply(Ad, _t(d * d), _t(z), u2)
            assert torch.equal(u1, u2)
    # gated launch is a no-op
    gate = torch.ones(1, dtype=torch.int32, device="cuda")
    u2.fill_(7.0)
    K.normal_apply(Ad, _t(d * d), _t(z), u2, gate=gate)
    assert bool((u2 == 7.0).all())
    # gemv / gemv_ratio / rhs with sub
    K.gemv(Ad, _t(x), u1, sub=_t(b))
    assert np.max(np.abs(_h(u1) - (A @ x - b))) <= 1e-13 * ((abs(A) @ x).max() + 1)
    K.gemv_ratio(Ad, _t(v), _t(s), u1)
    assert np.max(np.abs(_h(u1) - A @ (v / s))) <= 1e-13 * ((abs(A) @ abs(v / s)).max() + 1e-300)
    K.rhs(Ad, _t(x), _t(s), 0.3, u1, r_d=_t(c), r_p=_t(b))
    uu = (x - 0.3 / s) - (x / s) * c
    assert np.max(np.abs(_h(u1) - (A @ uu - b))) <= 1e-13 * ((abs(A) @ abs(uu)).max() + 1)
    # directions: elementwise outputs bit-identical to numpy given A'dy, A dx close
    ds, dx, atdy = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3))
    K.directions(Ad, _t(y), _t(x), _t(s), _t(v), 0.1, ds, dx, u1, atdy=atdy)
    assert np.max(np.abs(_h(atdy) - A.T @ y)) <= 1e-13 * ((abs(A.T) @ abs(y)).max() + 1)
    dsf = -_h(atdy)
    assert np.array_equal(_h(ds), dsf)
    assert np.array_equal(_h(dx), -x + 0.1 / s - (x / s) * dsf - v / s)
    assert np.max(np.abs(_h(u1) - A @ _h(dx))) <= 1e-12 * ((abs(A) @ abs(_h(dx))).max() + 1)
    # iterate: r_p = A x_new - b, r_d = A'y + s_new - c in one pass
    rp, rd = torch.empty(m, dtype=torch.float64, device="cuda"), torch.empty(
        n, dtype=torch.float64, device="cuda")
    xo, so = torch.empty_like(rd), torch.empty_like(rd)
    K.iterate(Ad, _t(x), _t(s), _t(y), _t(b), _t(c), rp, rd, dx=_t(v), ds=_t(v), alpha=0.5,
              x_out=xo, s_out=so)
    xn, sn = x + 0.5 * v, s + 0.5 * v
    assert np.array_equal(_h(xo), xn) and np.array_equal(_h(so), sn)
    assert np.max(np.abs(_h(rp) - (A @ xn - b))) <= 1e-13 * ((abs(A) @ abs(xn)).max() + 1)


def test_plan_not_applicable_falls_back_to_atomic_kernel(K):
    """A column of >= 1024 entries (or m > 65535) has no plan: the
    thread-per-column kernel runs, same results."""
    A = _ragged(4000, 2000, 9, maxlen=30)
    A = sp.hstack([A, sp.csc_matrix(np.ones((4000, 1)))]).tocsc()
    Ad = K.SparseDeviceMatrix.from_host(A)
    assert Ad.plan(force=True) == (None, 0)
    g = np.random.Generator(np.random.Philox(10))
    d2, z = g.random(A.shape[1]) + 0.5, g.standard_normal(4000)
    u = torch.empty(4000, dtype=torch.float64, device="cuda")
    K.normal_apply(Ad, _t(d2), _t(z), u)
    ref = A @ (d2 * (A.T @ z))
    assert np.max(np.abs(_h(u) - ref)) <= 1e-12 * np.abs(ref).max()
