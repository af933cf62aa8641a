"""Randomized bit-exactness sweep of the CSC sketch (large-m L2 kernel and both
bucket sorts) against the C restatement of scipy's order (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import torch
from oracle import chash
from oracle import ipm_oracle as O
from paper_2209_08722_b200 import sketching as S
from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram

rng = np.random.default_rng(int(os.environ.get("FUZZ_SEED", 1)))
bad = 0
for case in range(int(os.environ.get("FUZZ_N", 20))):
    m = int(rng.integers(2049, 4000))
    n = int(rng.integers(500, 6000))
    w = int(rng.integers(8, 900))
    s = int(rng.integers(1, 5))
    s = min(s, w)
    # nnz per column: 0 (empty), short, or long (up to 40)
    nnz = rng.choice([0, 1, 3, 5, 9, 17, 40], size=n, p=[.05, .15, .2, .3, .15, .1, .05])
    rows, cols, vals = [], [], []
    for j in range(n):
        r = rng.choice(m, size=int(nnz[j]), replace=False)
        rows.append(r); cols.append(np.full(r.size, j)); vals.append(rng.standard_normal(r.size))
    A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m, n))
    lp = DeviceLP.from_host(LinearProgram(A.tocsr(), np.zeros(m), np.ones(n)))
    d = 10.0 ** rng.uniform(-3, 3, n)
    seed = int(rng.integers(0, 1 << 30))
    W = S.build_sparse_embedding(n, w, s, seed)
    radix = case % 2 == 1
    if radix:
        os.environ["SKB_BUCKET_RADIX"] = "1"
    else:
        os.environ.pop("SKB_BUCKET_RADIX", None)
    X = S.apply_sketch(lp, torch.from_numpy(d).cuda(), W)
    cvals = O.sparse_embedding(n, w, s, seed)
    ref = chash.adw_dense(A.toarray(), d, cvals[0], cvals[1], w)
    got = X.cols[:, :m].cpu().numpy().T
    ok = np.array_equal(got, ref)
    bad += not ok
    print(f"case {case}: m={m} n={n} w={w} s={s} radix={radix} bit-exact={ok}", flush=True)
print("FAILURES", bad)
sys.exit(1 if bad else 0)
