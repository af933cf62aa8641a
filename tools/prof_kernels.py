"""One launch of each hot kernel at its config size, for `ncu -k regex:<name>`
captures (development aid). PROF_WHAT: k2 (c2 sketch apply s=1), syrk (c2 Gram
1000 x 1000 x 4000 lower), c3 (normal apply m=2000 n=1e6), c4 (CSC normal apply
m=1e4, 5 nnz/col, n=4e6)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200 import _lib
from paper_2209_08722_b200 import kernels as K
from paper_2209_08722_b200 import sketching as S
from paper_2209_08722_b200.lp_model import DeviceLP
from paper_2209_08722_b200.runtime import F64, lda_for, stream_ptr, workspace

what = os.environ.get("PROF_WHAT", "k2")
dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(0)


def dense(m, n):
    cols = torch.zeros((n, lda_for(m)), dtype=F64, device=dev)
    cols[:, :m].normal_(generator=g)
    return K.DeviceMatrix(cols, m)


if what == "k2":
    m, n = 1000, 1_000_000
    A = dense(m, n)
    lp = DeviceLP.from_device(A, torch.zeros(m, dtype=F64, device=dev),
                              torch.ones(n, dtype=F64, device=dev), n)
    d = torch.rand(n, dtype=F64, device=dev, generator=g) + 0.5
    W = S.build_sparse_embedding(n, 4000, 1, 5)
    for _ in range(2):
        S.apply_sketch(lp, d, W, check_positive=False)
elif what == "syrk":
    m, w = 1000, 4000
    X = torch.randn((w, m), dtype=F64, device=dev, generator=g)
    G = torch.zeros((1024, 1024), dtype=F64, device=dev)
    ws, cap = workspace(1 << 28)
    for _ in range(2):
        _lib.call("skb_gemm", 1, 0, m, m, w, 1.0, X, m, X, m, 0.0, G, 1024, 1, 1, 0, 0, 0, ws, cap,
                  stream_ptr())
elif what == "c3":
    m, n = 2000, 1_000_000
    A = dense(m, n)
    d2 = torch.rand(n, dtype=F64, device=dev, generator=g)
    z = torch.randn(m, dtype=F64, device=dev, generator=g)
    u = torch.empty(m, dtype=F64, device=dev)
    for _ in range(2):
        K.normal_apply(A, d2, z, u)
elif what == "c4":
    m, n, k = 10_000, 4_000_000, 5
    rows = torch.randint(0, m, (n, k), device=dev, generator=g, dtype=torch.int32)
    rows, _ = torch.sort(rows, dim=1)
    vals = torch.randn((n, k), dtype=F64, device=dev, generator=g)
    colptr = torch.arange(0, n * k + 1, k, dtype=torch.int64, device=dev)
    A = K.SparseDeviceMatrix(colptr, rows.reshape(-1).contiguous(), vals.reshape(-1), m)
    d2 = torch.rand(n, dtype=F64, device=dev, generator=g)
    z = torch.randn(m, dtype=F64, device=dev, generator=g)
    u = torch.empty(m, dtype=F64, device=dev)
    for _ in range(2):
        K.normal_apply(A, d2, z, u)
torch.cuda.synchronize()
print("ok", what)
