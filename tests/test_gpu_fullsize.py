"""BASELINE full-size configurations on the B200, checked through properties
that do not need the CPU oracle (which cannot hold c3/c4): agreement with an
independent cuBLAS / cuSPARSE fp64 evaluation of the same formula (different
summation order: 1e-12 relative), linearity and symmetry of the normal
operator, bucket sums of the sketch, and the factor's defining identity."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _dense(dev, m, n, seed):
    from paper_2209_08722_b200 import kernels as K
    from paper_2209_08722_b200.runtime import F64, lda_for
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev)
    cols[:, :m].normal_(generator=g)
    d2 = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.1
    return K.DeviceMatrix(cols, m), d2, g


def _check_normal(K, A, d2, g, ref_fn, m):
    from paper_2209_08722_b200.runtime import F64
    z1 = torch.randn(m, dtype=F64, device=A.cols.device if hasattr(A, "cols") else "cuda",
                     generator=g)
    z2 = torch.randn_like(z1)
    u1, u2, u3 = (torch.empty_like(z1) for _ in range(3))
    K.normal_apply(A, d2, z1, u1)
    K.normal_apply(A, d2, z2, u2)
    K.normal_apply(A, d2, 0.75 * z1 - 2.0 * z2, u3)
    ref = ref_fn(z1)
    scale = ref.abs().max().item()
    assert (u1 - ref).abs().max().item() <= 1e-12 * scale              # independent evaluation
    lin = 0.75 * u1 - 2.0 * u2
    assert (u3 - lin).abs().max().item() <= 1e-12 * lin.abs().max().item()   # linearity
    s12, s21 = torch.dot(z1, u2).item(), torch.dot(u1, z2).item()
    assert abs(s12 - s21) <= 1e-11 * max(abs(s12), 1.0)                  # symmetry
    assert torch.dot(z1, u1).item() > 0                                  # positive definite


def test_c2_normal_operator_fullsize(dev):
    from paper_2209_08722_b200 import kernels as K
    m, n = 1000, 1_000_000
    A, d2, g = _dense(dev, m, n, 21)
    At = A.cols[:, :m]                       # n x m view: A' (column j of A is row j here)
    _check_normal(K, A, d2, g, lambda z: At.t() @ (d2 * (At @ z)), m)


def test_c3_normal_operator_fullsize(dev):
    from paper_2209_08722_b200 import kernels as K
    m, n = 2000, 4_000_000                   # 64 GB: the sharded config on one GPU
    A, d2, g = _dense(dev, m, n, 23)
    At = A.cols[:, :m]
    _check_normal(K, A, d2, g, lambda z: At.t() @ (d2 * (At @ z)), m)
    del A, At
    torch.cuda.empty_cache()


def test_c4_sparse_normal_operator_fullsize(dev):
    from paper_2209_08722_b200 import kernels as K
    from paper_2209_08722_b200.runtime import F64
    m, n, k = 10_000, 20_000_000, 5
    g = torch.Generator(device=dev)
    g.manual_seed(24)
    rows = torch.randint(0, m, (n, k), device=dev, generator=g, dtype=torch.int64)
    rows, _ = torch.sort(rows, dim=1)
    vals = torch.randn((n, k), dtype=F64, device=dev, generator=g)
    colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device=dev)
    A = K.SparseDeviceMatrix(colptr, rows.to(torch.int32).reshape(-1).contiguous(),
                             vals.reshape(-1), m)
    d2 = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.1
    cidx = torch.arange(n, device=dev).repeat_interleave(k)
    S = torch.sparse_coo_tensor(torch.stack([rows.reshape(-1), cidx]), vals.reshape(-1),
                                (m, n)).coalesce()
    St = S.t().coalesce()
    ref_fn = lambda z: torch.sparse.mm(S, (d2 * torch.sparse.mm(St, z[:, None])[:, 0])[:, None])[:, 0]  # noqa: E731
    _check_normal(K, A, d2, g, ref_fn, m)


def test_c2_sketch_and_factor_fullsize(dev):
    """ADW (s = 1, w = 4000) bucket sums against an index_add evaluation, and
    the CholeskyQR2 factor: Linv (X'X) Linv' = I and apply_inv = Q^-1."""
    from paper_2209_08722_b200 import preconditioning as PC
    from paper_2209_08722_b200 import sketching as S
    from paper_2209_08722_b200.lp_model import DeviceLP
    from paper_2209_08722_b200.runtime import F64
    m, n, w = 1000, 1_000_000, 4000
    A, d2, g = _dense(dev, m, n, 25)
    d = d2.sqrt()
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=dev),
                              torch.ones(n, dtype=F64, device=dev), n)
    W = S.build_sparse_embedding(n, w, 1, 77)
    X = S.apply_sketch(lp, d, W, check_positive=False)
    Xh = X.cols[:, :m]
    At = A.cols[:, :m]
    ref = torch.zeros((w, m), dtype=F64, device=dev)
    ref.index_add_(0, W.cols[:, 0].long(), At * (d * W.vals[:, 0])[:, None])
    scale = (At.abs() * d[:, None]).sum(0).max().item()
    assert (Xh - ref).abs().max().item() <= 1e-13 * scale
    f = PC.build_preconditioner(X)
    Q = Xh.t() @ Xh
    Li = f.Linv[:m, :m]
    E = Li @ Q @ Li.t() - torch.eye(m, dtype=F64, device=dev)
    assert E.abs().max().item() <= 1e-10
    r = torch.randn(m, dtype=F64, device=dev, generator=g)
    z = PC.apply_inv(f, r)
    assert ((Q @ z) - r).abs().max().item() <= 1e-9 * r.abs().max().item() * math.sqrt(m)
    assert np.isfinite(f.diag_min) and f.diag_min > 0
