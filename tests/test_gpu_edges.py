"""Edge cases the reference's own tests exercise (reference tests/test_sketching.py,
test_preconditioning.py, test_krylov_solvers.py, test_lp_model.py), run through
the device API: tiny and ragged shapes, invalid dimensions, error classes,
determinism, and agreement with dense products."""

import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import ipm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _h(t):
    return t.detach().cpu().numpy()


def _dense_sketch(W):
    if W.kind == "identity":
        return np.eye(W.n)
    if W.kind == "gaussian":
        return _h(W.dense)
    D = np.zeros((W.n, W.w))
    cols, vals = _h(W.cols), _h(W.vals)
    for j in range(W.n):
        D[j, cols[j]] = vals[j]
    return D


def _random_lp(m, n, density, seed):
    g = np.random.Generator(np.random.Philox(seed))
    A = np.where(g.random((m, n)) < density, g.standard_normal((m, n)), 0.0)
    A[np.arange(m), np.arange(m) % n] += 1.0   # no zero rows
    return A


def _device_lp(A):
    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    m, n = A.shape
    return DeviceLP.from_host(LinearProgram(sp.csr_matrix(A), np.ones(m), np.ones(n)))


# ------------------------------------------------------------- sketches
@pytest.mark.parametrize("n,w,s,seed", [(1, 1, 1, 0), (7, 7, 1, 1), (12, 8, 2, 4), (50, 24, 3, 9),
                                        (10, 4, 4, 2), (200, 3, 1, 5), (33, 64, 2, 6)])
def test_sparse_embedding_rows(dev, n, w, s, seed):
    """Exactly s distinct buckets per row, values +-1/sqrt(s), equal to the oracle."""
    from paper_2209_08722_b200 import sketching as S
    W = S.build_sparse_embedding(n, w, s, seed)
    D = _dense_sketch(W)
    assert np.all(np.count_nonzero(D, axis=1) == s)
    assert np.allclose(np.abs(D[D != 0.0]), 1.0 / math.sqrt(s))
    cols, vals = O.sparse_embedding(n, w, s, seed)
    assert np.array_equal(_h(W.cols), cols) and np.array_equal(_h(W.vals), vals)
    W2 = S.build_sparse_embedding(n, w, s, seed)
    assert np.array_equal(_h(W.cols), _h(W2.cols))
    u = np.arange(float(w))
    assert np.allclose(_h(W.matvec(_t(u))), D @ u, atol=1e-14)


def test_as_sparse_matches_reference_layout(dev):
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.errors import DimensionMismatch
    W = S.build_sparse_embedding(50, 24, 3, 9)
    csr = W.as_sparse()
    cols, vals = O.sparse_embedding(50, 24, 3, 9)
    D = np.zeros((50, 24))
    for j in range(50):
        D[j, cols[j]] = vals[j]
    assert np.array_equal(csr.toarray(), D) and csr.has_sorted_indices
    assert np.array_equal(S.build_identity_sketch(4).as_sparse().toarray(), np.eye(4))
    with pytest.raises(DimensionMismatch):
        S.build_gaussian_sketch(10, 3, 1).as_sparse()


def test_sketch_invalid_dims(dev):
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.errors import InvalidDims
    with pytest.raises(InvalidDims):
        S.build_sparse_embedding(10, 4, 5, 0)      # s > w
    with pytest.raises(InvalidDims):
        S.build_sparse_embedding(2, 10, 2, 0)      # w > n s
    with pytest.raises(InvalidDims):
        S.build_sparse_embedding(10, 4, 0, 0)      # s < 1
    with pytest.raises(InvalidDims):
        S.build_gaussian_sketch(10, 0, 0)
    with pytest.raises(InvalidDims):
        S.build_identity_sketch(0)


def test_gaussian_and_identity_small(dev):
    from paper_2209_08722_b200 import sketching as S
    W = S.build_gaussian_sketch(30, 10, 2)
    assert np.array_equal(_h(W.dense), _h(S.build_gaussian_sketch(30, 10, 2).dense))
    assert np.array_equal(_h(W.dense), O.gaussian_sketch(30, 10, 2))
    I = S.build_identity_sketch(5)
    assert np.array_equal(_h(I.matvec(_t(np.arange(5.0)))), np.arange(5.0))


@pytest.mark.parametrize("kind", ["sparse", "gaussian", "identity"])
@pytest.mark.parametrize("m,extra,seed", [(1, 0, 1), (1, 5, 2), (3, 0, 3), (5, 20, 4), (8, 3, 5),
                                          (2, 13, 6)])
def test_apply_sketch_matches_dense_triple_product(dev, kind, m, extra, seed):
    from paper_2209_08722_b200 import sketching as S
    n = m + extra
    A = _random_lp(m, n, 0.5, seed)
    lp = _device_lp(A)
    d = np.random.Generator(np.random.Philox(seed + 1)).random(n) + 0.1
    w = max(1, min(n, m + 2))
    if kind == "gaussian":
        W = S.build_gaussian_sketch(n, w, seed + 2)
    elif kind == "identity":
        W = S.build_identity_sketch(n)
    else:
        W = S.build_sparse_embedding(n, w, min(2, w), seed + 2)
    X = S.apply_sketch(lp, _t(d), W)
    out = _h(X.cols)[:, :m].T
    ref = A @ np.diag(d) @ _dense_sketch(W)
    assert np.max(np.abs(out - ref)) <= 1e-12 * max(1.0, np.abs(ref).max())


def test_apply_sketch_errors(dev):
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.errors import DimensionMismatch, NonpositiveScaling
    lp = _device_lp(_random_lp(3, 6, 0.5, 0))
    W = S.build_gaussian_sketch(6, 4, 0)
    with pytest.raises(DimensionMismatch):
        S.apply_sketch(lp, _t(np.ones(5)), W)
    with pytest.raises(NonpositiveScaling):
        S.apply_sketch(lp, _t(np.zeros(6)), W)
    with pytest.raises(DimensionMismatch):
        S.apply_sketch(lp, _t(np.ones(6)), S.build_gaussian_sketch(7, 4, 0))


def test_permutation_sketch_is_column_permutation(dev):
    from paper_2209_08722_b200 import sketching as S
    A = _random_lp(4, 10, 0.5, 0)
    lp = _device_lp(A)
    perm = np.random.Generator(np.random.Philox(3)).permutation(10)
    W = S.SketchOperator(kind="sparse_sign", n=10, w=10, s=1, seed=0,
                         cols=torch.from_numpy(perm.astype(np.int32)).reshape(10, 1).cuda(),
                         vals=torch.ones((10, 1), dtype=torch.float64, device="cuda"))
    X = _h(S.apply_sketch(lp, _t(np.ones(10)), W).cols)[:, :4].T
    expect = np.zeros_like(A)
    for i, j in enumerate(perm):
        expect[:, j] = A[:, i]
    assert np.array_equal(X, expect)


# -------------------------------------------------------- preconditioner
def test_preconditioner_errors_and_identity_sketch(dev):
    from paper_2209_08722_b200 import preconditioning as PC
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.errors import RankDeficient
    from paper_2209_08722_b200.kernels import DeviceMatrix
    g = np.random.Generator(np.random.Philox(3))
    X = DeviceMatrix(_t(g.standard_normal((3, 6))), 5)            # w = 3 < m = 5
    with pytest.raises(RankDeficient):
        PC.build_preconditioner(X)
    # full-row-rank ADW with the identity sketch (w = n): Q^-1 exact
    A = _random_lp(6, 9, 0.7, 1)
    lp = _device_lp(A)
    d = g.random(9) + 0.5
    Xd = S.apply_sketch(lp, _t(d), S.build_identity_sketch(9))
    f = PC.build_preconditioner(Xd)
    r = g.standard_normal(6)
    Q = A @ np.diag(d * d) @ A.T
    assert np.allclose(_h(PC.apply_inv(f, _t(r))), np.linalg.solve(Q, r), rtol=1e-10, atol=0)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 37), (2, 3), (31, 33), (63, 64), (65, 130),
                                 (129, 1000), (1023, 1024), (1025, 1200)])
def test_ragged_normal_operator(dev, m, n):
    """Shapes around the warp / tile / padding boundaries."""
    from paper_2209_08722_b200.krylov_solvers import NormalOperator
    A = _random_lp(m, n, 1.0, m * 7 + n)
    lp = _device_lp(A)
    d = np.random.Generator(np.random.Philox(n)).random(n) + 0.1
    z = np.random.Generator(np.random.Philox(m)).standard_normal(m)
    op = NormalOperator(lp, _t(d))
    ref = A @ (d * d * (A.T @ z))
    scale = np.abs(A) @ (d * d * (np.abs(A.T) @ np.abs(z)))
    assert np.max(np.abs(_h(op.apply(_t(z))) - ref) / np.maximum(scale, 1e-300)) <= 1e-13


def test_lp_validation(dev):
    from paper_2209_08722_b200.errors import DimensionMismatch, ZeroRow
    from paper_2209_08722_b200.lp_model import make_lp
    with pytest.raises(DimensionMismatch):
        make_lp(np.ones((3, 2)), np.ones(3), np.ones(2))            # n < m
    A = np.ones((2, 4))
    A[1] = 0.0
    with pytest.raises(ZeroRow):
        make_lp(A, np.ones(2), np.ones(4))
    with pytest.raises(DimensionMismatch):
        make_lp(np.ones((2, 4)), np.ones(3), np.ones(4))
    with pytest.raises(ValueError):
        make_lp(np.full((2, 4), np.nan), np.ones(2), np.ones(4))
