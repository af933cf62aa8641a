"""Sparse A (CSC on the device, config c4): kernels, bit-exact ADW, trajectory."""

import hashlib
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN
from oracle import chash
from oracle import ipm_oracle as O
from paper_2209_08722_b200.problems import sparse_wide_lp

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


@pytest.mark.parametrize("m,n,k", [(100, 20_000, 5), (1000, 50_000, 5), (10_000, 200_000, 5),
                                   (37, 3000, 3)])
def test_csc_passes(K, m, n, k):
    lpd = sparse_wide_lp(m, n, k, 3)
    A = lpd.A
    g = np.random.Generator(np.random.Philox(4))
    d = 10.0 ** g.uniform(-2, 2, n)
    z, y, b = g.standard_normal(m), g.standard_normal(m), g.standard_normal(m)
    x, s, c = g.random(n) + 0.2, g.random(n) + 0.2, g.standard_normal(n)
    Ad = K.SparseDeviceMatrix.from_host(A)
    u = torch.empty(m, dtype=torch.float64, device="cuda")
    K.normal_apply(Ad, _t(d * d), _t(z), u)
    ref = A @ (d * d * (A.T @ z))
    scale = abs(A) @ (d * d * (abs(A.T) @ abs(z)))
    assert np.max(np.abs(_h(u) - ref) / scale) <= 1e-13
    K.gemv(Ad, _t(x), u, sub=_t(b))
    assert np.max(np.abs(_h(u) - (A @ x - b))) <= 1e-13 * (abs(A) @ x).max()
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    K.gemv_t(Ad, _t(y), t, add=_t(s), sub=_t(c))
    assert np.max(np.abs(_h(t) - (A.T @ y + s - c))) <= 1e-13 * (abs(A.T) @ abs(y) + 1).max()
    ds, dx, atdy = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3))
    adx = torch.empty(m, dtype=torch.float64, device="cuda")
    v = 1e-3 * g.standard_normal(n)
    K.directions(Ad, _t(y), _t(x), _t(s), _t(v), 0.1, ds, dx, adx, atdy=atdy)
    Aty = A.T @ y
    assert np.max(np.abs(_h(atdy) - Aty)) <= 1e-13 * (abs(A.T) @ abs(y)).max()
    ds_from = -_h(atdy)
    assert np.array_equal(_h(ds), ds_from)
    assert np.array_equal(_h(dx), -x + 0.1 / s - (x / s) * ds_from - v / s)
    assert np.max(np.abs(_h(adx) - A @ _h(dx))) <= 1e-12 * (abs(A) @ abs(_h(dx))).max()


def test_csc_sketch_apply_bit_exact(K):
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    with open(os.path.join(GOLDEN, "sparse_traces.json")) as f:
        gold = json.load(f)
    lpd = sparse_wide_lp(100, 20_000, 5, 7)
    lp = DeviceLP.from_host(LinearProgram(lpd.A.tocsr(), lpd.b, lpd.c))
    assert lp.sparse
    d = 10.0 ** np.random.Generator(np.random.Philox(78)).uniform(-3, 3, lpd.n)
    W = S.build_sparse_embedding(lpd.n, 400, 4, 77)
    X = S.apply_sketch(lp, _t(d), W)
    adw = np.ascontiguousarray(_h(X.cols)[:, :100].T)
    assert hashlib.sha256(adw.tobytes()).hexdigest() == gold["adw_sha256"]
    # and against the C restatement of scipy's summation order, s = 1, larger m
    lpd = sparse_wide_lp(3000, 50_000, 5, 8)
    lp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c))
    d = 10.0 ** np.random.Generator(np.random.Philox(79)).uniform(-3, 3, lpd.n)
    W = S.build_sparse_embedding(lpd.n, 6000, 1, 80)
    X = S.apply_sketch(lp, _t(d), W)
    cols, vals = O.sparse_embedding(lpd.n, 6000, 1, 80)
    ref = chash.adw_dense(lpd.A.toarray(), d, cols, vals, 6000)
    assert np.array_equal(_h(X.cols)[:, :3000].T, ref)


@pytest.mark.parametrize("kernel", ["ell", "bids", "l2"])
@pytest.mark.parametrize("m,n,k,w,s,radix", [(2500, 10_000, 5, 600, 4, False),
                                              (2600, 8000, 12, 500, 3, False),
                                              (2500, 10_000, 5, 600, 4, True),
                                              (2500, 10_000, 0, 700, 4, False),
                                              (2500, 20_000, 5, 4, 2, False),
                                              (2500, 20_000, 0, 3, 2, False),
                                              (20_000, 2000, 5, 50, 4, False),
                                              (30_000, 1000, 5, 40, 1, False)])
def test_csc_sketch_large_m_bit_exact(K, monkeypatch, m, n, k, w, s, radix, kernel):
    """m > 2048 takes the warp-per-bucket L2 kernel: few buckets (many repeated
    rows per member chunk -> the ordered path) and columns longer than its
    8-entry register window (k = 12 -> the lane-by-lane path), bit-exact
    against the C restatement of scipy's summation order. radix: the bucket
    order from the CUB radix sort (its default from 2^20 entries, forced here)
    instead of the counting sort. kernel: the ELL-record kernel (one CTA per
    bucket, rows binned to owner warps; k = 0: ragged columns of 0..12 entries, the
    long ones split a batch), its bid-round variant (SKB_CSC_SKETCH_BIDS=1) or the L2
    kernel (SKB_CSC_SKETCH_L2=1). w = 3-4: 1e4+ members per bucket, several chunks of the
    row-sorting kernel (later chunks continue each row from X). m = 2e4 / 3e4: past the
    bid-round kernel's (and at 3e4 the row-sorting kernel's) shared-memory ceiling, where
    the dispatch falls back to the next kernel that fits."""
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    if radix:
        monkeypatch.setenv("SKB_BUCKET_RADIX", "1")
    if kernel == "l2":
        monkeypatch.setenv("SKB_CSC_SKETCH_L2", "1")
    if kernel == "bids":
        monkeypatch.setenv("SKB_CSC_SKETCH_BIDS", "1")
    if k == 0:  # ragged: mostly short columns, some longer than an ELL record
        g0 = np.random.Generator(np.random.Philox(m + n))
        lens = np.where(g0.random(n) < 0.9, g0.integers(0, 6, n), g0.integers(6, 13, n))
        rows = [np.sort(g0.choice(m, size=int(c), replace=False)) for c in lens]
        ptr = np.concatenate([[0], np.cumsum(lens)])
        Asp = sp.csc_matrix((g0.standard_normal(int(ptr[-1])), np.concatenate(rows), ptr),
                            shape=(m, n))
        lpd = sparse_wide_lp(m, n, 5, m)
        lpd.A = Asp
    else:
        lpd = sparse_wide_lp(m, n, k, m + k)
    lp = DeviceLP.from_host(LinearProgram(lpd.A, lpd.b, lpd.c))
    assert (lp.A.ell() is not None)
    d = 10.0 ** np.random.Generator(np.random.Philox(m)).uniform(-3, 3, lpd.n)
    W = S.build_sparse_embedding(lpd.n, w, s, 90 + k)
    X = S.apply_sketch(lp, _t(d), W)
    cols, vals = O.sparse_embedding(lpd.n, w, s, 90 + k)
    ref = chash.adw_dense(lpd.A.toarray(), d, cols, vals, w)
    assert np.array_equal(_h(X.cols)[:, :m].T, ref)


@pytest.mark.parametrize("planned", ["0", "1"])
def test_sparse_trajectory_s4(K, monkeypatch, planned):
    """planned=1: every m-vector A-pass on the deterministic planned kernel."""
    monkeypatch.setenv("SKB_CSC_PLAN", planned)
    from paper_2209_08722_b200 import ipm_core as IC
    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    with open(os.path.join(GOLDEN, "sparse_traces.json")) as f:
        gold = json.load(f)["s4"]
    lpd = sparse_wide_lp(100, 20_000, 5, 7)
    dlp = DeviceLP.from_host(LinearProgram(lpd.A.tocsr(), lpd.b, lpd.c))
    assert dlp.sparse
    assert (dlp.A.plan()[0] is not None) == (planned == "1")
    kw = dict(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=400, s=4, tol_outer=1e-6,
              seed=11)
    rep = IC.solve(dlp, IC.make_iterate(dlp, lpd.x0, lpd.y0, lpd.s0), IC.IpmParams(**kw))
    # reference floor: same algorithm, normal operator summed in another order
    A = sp.csr_matrix(lpd.A)
    Ad = lpd.A.toarray()
    monkeypatch.setattr(O.NormalOp, "apply", lambda self, v: Ad @ (self.d2 * (Ad.T @ v)))
    ref = O.solve(A, lpd.b, lpd.c, O.make_iterate(A, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0),
                  O.Params(**kw))
    assert rep.outer == gold["outer"]
    assert [r.inner_iterations for r in rep.steps] == gold["inner_iterations"]
    assert [r.sketch_seed for r in rep.steps] == [s["sketch_seed"] for s in gold["steps"]]
    floor = np.maximum.accumulate(np.abs(np.array(ref["mu_trace"]) - np.array(gold["mu_trace"])) /
                                  np.array(gold["mu_trace"]))
    dev = np.abs(np.array(rep.mu_trace) - np.array(gold["mu_trace"])) / np.array(gold["mu_trace"])
    assert np.all(dev <= np.maximum(1e-9, 4 * floor)), (dev, floor)
    assert abs(rep.objective - gold["objective"]) <= 1e-8 * abs(gold["objective"])


@pytest.mark.parametrize("m", [20_000, 40_000])
def test_csc_passes_past_shared_memory_ceiling(K, m):
    """m past the shared-memory CSC kernels' ceiling (z and the partial m-vector:
    m <= 14,080; one vector: m <= 28,160): the global-memory pass. Normal operator,
    A x - sub and A'y against scipy."""
    from paper_2209_08722_b200.kernels import SparseDeviceMatrix
    g = np.random.Generator(np.random.Philox(m))
    n = 3 * m
    rows = np.stack([g.choice(m, size=5, replace=False) for _ in range(n)])
    A = sp.csc_matrix((g.standard_normal(5 * n), rows.reshape(-1), np.arange(0, 5 * n + 1, 5)),
                      shape=(m, n))
    Ad = SparseDeviceMatrix.from_host(A)
    d2 = 10.0 ** g.uniform(-2, 2, n)
    z, x, y = g.standard_normal(m), g.standard_normal(n), g.standard_normal(m)
    sub = g.standard_normal(m)
    u = torch.empty(m, dtype=torch.float64, device="cuda")
    K.normal_apply(Ad, _t(d2), _t(z), u, sub=_t(sub))
    ref = A @ (d2 * (A.T @ z)) - sub
    scale = (abs(A) @ (d2 * (abs(A.T) @ abs(z)))).max()
    assert np.max(np.abs(_h(u) - ref)) <= 1e-13 * scale
    K.gemv(Ad, _t(x), u)
    assert np.max(np.abs(_h(u) - A @ x)) <= 1e-13 * (abs(A) @ abs(x)).max()
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    K.gemv_t(Ad, _t(y), t)
    assert np.max(np.abs(_h(t) - A.T @ y)) <= 1e-13 * (abs(A.T) @ abs(y)).max()
