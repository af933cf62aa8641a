"""Generate the golden fixtures under tests/golden/ from the LIVE reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

The fixtures pin the oracle (oracle/) to the reference; the GPU parity tests
then compare the CUDA path with the oracle on the box, where the reference is
absent. Outputs are small: hash tables, checksums, ADW bits, traces.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

import skipm  # noqa: E402
from skipm import ipm_core, krylov_solvers, preconditioning, sketching  # noqa: E402

from paper_2209_08722_b200.problems import wide_dense_lp  # noqa: E402

# (n, w, s, seed): s=1 CountSketch, Lemire rejections at large w, duplicate
# redraws at s>1, and the 2s >= w argsort branch.
HASH_CASES = [
    (10_000, 400, 1, 11), (20_000, 4_000, 1, 12), (5_000, 3, 1, 13),
    (3_000, 400, 18, 14), (2_000, 4_000, 20, 15), (500, 64, 8, 16),
    (1_000, 40, 4, 17), (30, 8, 5, 18), (64, 12, 6, 19), (7, 7, 1, 20),
    (1, 1, 1, 22),
]
BIG_HASH_CASES = [(1_000_000, 4_000, 1, 31), (1_000_000, 4_000, 4, 32),
                  (4_000_000, 8_000, 1, 33),
                  (20_000_000, 40_000, 4, 34),  # config c4 at s = 4 (the parity setting)
                  (4_000_000, 8_000, 4, 35)]    # config c3 at s = 4


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hashes():
    out = {}
    for (n, w, s, seed) in HASH_CASES:
        W = sketching.build_sparse_embedding(n, w, s, seed)
        key = f"{n}_{w}_{s}_{seed}"
        out[f"cols_{key}"] = W.cols.astype(np.int64)
        out[f"sign_{key}"] = (W.vals > 0).astype(np.int8)
    # raw bounded draws with a high Lemire rejection rate (threshold 2^30)
    for w in (3 * 2**30, 2**31 + 1, 5):
        g = np.random.Generator(np.random.Philox(21))
        out[f"lemire_{w}"] = g.integers(0, w, size=4000)
    np.savez_compressed(os.path.join(HERE, "hashes.npz"), **out)
    big = []
    for (n, w, s, seed) in BIG_HASH_CASES:
        W = sketching.build_sparse_embedding(n, w, s, seed)
        big.append(dict(n=n, w=w, s=s, seed=seed,
                        cols_sha256=sha(W.cols.astype(np.int64)),
                        sign_sha256=sha((W.vals > 0).astype(np.int8)),
                        cols_head=W.cols[:4].tolist(), cols_tail=W.cols[-4:].tolist()))
    seeds = {}
    for seed in (0, 1, 7, 12345):
        g = np.random.Generator(np.random.Philox(seed))
        key = np.random.SeedSequence(seed).generate_state(2, np.uint64)
        seeds[str(seed)] = dict(key=[int(k) for k in key],
                                draws=[int(g.integers(0, 2**63)) for _ in range(8)])
    with open(os.path.join(HERE, "hashes_big.json"), "w") as f:
        json.dump(dict(big=big, outer_seeds=seeds), f, indent=1)


def adw():
    out = {}
    g = np.random.Generator(np.random.Philox(99))
    m, n = 20, 600
    A = g.standard_normal((m, n))
    d = 10.0 ** g.uniform(-2, 1, n)
    out["A"], out["d"] = A, d
    lp = skipm.make_lp(A, np.zeros(m), np.ones(n))
    for s in (1, 4):
        W = sketching.build_sparse_embedding(n, 64, s, 100 + s)
        out[f"adw_s{s}"] = sketching.apply_sketch(lp.A, d, W)
        out[f"seed_s{s}"] = np.array(100 + s)
    # normal operator and preconditioned CG on the same data
    W = sketching.build_sparse_embedding(n, 64, 4, 104)
    f = preconditioning.build_preconditioner(sketching.apply_sketch(lp.A, d, W),
                                             sketch_tag=W.tag)
    op = krylov_solvers.NormalOperator(lp.A, d)
    v = g.standard_normal(m)
    out["v"], out["normal_apply"] = v, op.apply(v)
    dy, tr = krylov_solvers.pcg(op, f, v, 30, 1e-10)
    out["pcg_dy"], out["pcg_norms"] = dy, np.array(tr.residual_norms)
    out["inv_v"] = preconditioning.apply_inv(f, v)
    out["pinv_v"] = preconditioning.apply_pinv_adw(f, v)
    np.savez_compressed(os.path.join(HERE, "adw_small.npz"), **out)


def c1_traces():
    res = {}
    lpd = wide_dense_lp(100, 10_000, 0)
    lp = skipm.make_lp(lpd.A, lpd.b, lpd.c, name=lpd.name)
    gamma = lpd.gamma_run(0.1)
    for s_nnz in (4, 1):
        start = ipm_core.make_iterate(lp, lpd.x0, lpd.y0, lpd.s0)
        prm = ipm_core.IpmParams(mode="feasible", gamma=gamma, sigma=0.5, sketch="sparse",
                                 w=400, s=s_nnz, tol_outer=1e-6, seed=0)
        rep = ipm_core.solve(lp, start, prm)
        d = rep.to_dict()
        d.pop("params")
        d["x_sha256"] = sha(rep.x)
        d["x_head"] = rep.x[:8].tolist()
        d["y"] = rep.y.tolist()
        res[f"s{s_nnz}"] = d
        print(f"c1 s={s_nnz}: outer {rep.outer} inner {rep.sum_inner} obj {rep.objective!r}")
    res["gamma_run"] = gamma
    with open(os.path.join(HERE, "c1_traces.json"), "w") as f:
        json.dump(res, f)


def small_traces():
    """A smaller LP (m=40, n=3000) in both modes, for fast lock-step checks."""
    res = {}
    lpd = wide_dense_lp(40, 3000, 5)
    lp = skipm.make_lp(lpd.A, lpd.b, lpd.c, name=lpd.name)
    for mode in ("feasible", "infeasible"):
        start = ipm_core.make_iterate(lp, lpd.x0, lpd.y0, lpd.s0)
        if mode == "feasible":
            prm = ipm_core.IpmParams(mode=mode, gamma=lpd.gamma_run(0.1), sigma=0.5, w=160,
                                     s=4, tol_outer=1e-7, seed=3)
        else:
            start = ipm_core.make_iterate(lp, np.ones(lp.n), np.zeros(lp.m), np.ones(lp.n))
            prm = ipm_core.IpmParams(mode=mode, gamma=0.5, sigma=0.5, w=160, s=4,
                                     tol_outer=1e-7, seed=4, max_outer=60)
        try:
            rep = ipm_core.solve(lp, start, prm)
        except skipm.MaxIterations as e:
            rep = e.report
        d = rep.to_dict()
        d.pop("params")
        res[mode] = d
        print(f"small {mode}: outer {rep.outer} conv {rep.converged} obj {rep.objective!r}")
    with open(os.path.join(HERE, "small_traces.json"), "w") as f:
        json.dump(res, f)


def solver_traces():
    """The other inner solvers (krylov_solvers.py:108-204) and correction off, on the
    small LP in feasible mode (ipm_core.py:436-456)."""
    res = {}
    lpd = wide_dense_lp(40, 3000, 5)
    lp = skipm.make_lp(lpd.A, lpd.b, lpd.c, name=lpd.name)
    # Chebyshev's fixed band needs a certified embedding: w = 1200, s = 12 (at w = 4m it
    # stalls for 200 outer steps in the reference too).
    cases = {"chebyshev": dict(solver="chebyshev", w=1200, s=12),
             "unpreconditioned": dict(solver="unpreconditioned", w=160, s=4),
             "direct": dict(solver="direct", w=160, s=4),
             "pcg_nocorr": dict(solver="pcg", correction=False, w=160, s=4)}
    for name, kw in cases.items():
        start = ipm_core.make_iterate(lp, lpd.x0, lpd.y0, lpd.s0)
        prm = ipm_core.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5,
                                 tol_outer=1e-6, seed=5, **kw)
        try:
            rep = ipm_core.solve(lp, start, prm)
        except skipm.MaxIterations as e:
            rep = e.report
        d = rep.to_dict()
        d.pop("params")
        res[name] = d
        print(f"{name}: outer {rep.outer} conv {rep.converged} inner {rep.sum_inner} "
              f"obj {rep.objective!r}")
    with open(os.path.join(HERE, "solver_traces.json"), "w") as f:
        json.dump(res, f)


def gaussian_traces():
    """build_gaussian_sketch values (sketching.py:131-139) and Gaussian-sketch solves,
    incl. the ill-conditioned c5 generator (repaired start)."""
    from paper_2209_08722_b200.problems import ill_conditioned_lp
    res = {"sketch": []}
    for (n, w, seed) in [(3000, 64, 41), (100_000, 40, 42), (7, 3, 43)]:
        W = sketching.build_gaussian_sketch(n, w, seed)
        res["sketch"].append(dict(n=n, w=w, seed=seed, sha256=sha(W.dense),
                                  head=W.dense.ravel()[:6].tolist(),
                                  tail=W.dense.ravel()[-6:].tolist()))
    for name, lpd in [("wide", wide_dense_lp(40, 3000, 5)), ("illcond", ill_conditioned_lp(30, 2000, 6))]:
        lp = skipm.make_lp(lpd.A, lpd.b, lpd.c, name=lpd.name)
        start = ipm_core.make_iterate(lp, lpd.x0, lpd.y0, lpd.s0)
        prm = ipm_core.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1),
                                 sigma=0.5 if name == "wide" else 0.3, sketch="gaussian",
                                 w=4 * lpd.m, tol_outer=1e-6, seed=9)
        rep = ipm_core.solve(lp, start, prm)
        d = rep.to_dict()
        d.pop("params")
        res[name] = d
        print(f"gaussian {name}: outer {rep.outer} inner {rep.sum_inner} obj {rep.objective!r}")
    with open(os.path.join(HERE, "gaussian_traces.json"), "w") as f:
        json.dump(res, f)


def sparse_traces():
    """Config c4's generator at reduced size (5 nnz per column), s = 4 and s = 1."""
    from paper_2209_08722_b200.problems import sparse_wide_lp
    res = {}
    lpd = sparse_wide_lp(100, 20_000, 5, 7)
    lp = skipm.make_lp(lpd.A, lpd.b, lpd.c, name=lpd.name)
    for s_nnz in (4, 1):
        start = ipm_core.make_iterate(lp, lpd.x0, lpd.y0, lpd.s0)
        prm = ipm_core.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=400,
                                 s=s_nnz, tol_outer=1e-6, seed=11)
        rep = ipm_core.solve(lp, start, prm)
        d = rep.to_dict()
        d.pop("params")
        res[f"s{s_nnz}"] = d
        print(f"sparse s={s_nnz}: outer {rep.outer} inner {rep.sum_inner} obj {rep.objective!r}")
    # ADW bits for the CSC sketch kernel
    W = sketching.build_sparse_embedding(lpd.n, 400, 4, 77)
    g = np.random.Generator(np.random.Philox(78))
    d = 10.0 ** g.uniform(-3, 3, lpd.n)
    adw = sketching.apply_sketch(lp.A, d, W)
    res["adw_sha256"] = sha(adw)
    with open(os.path.join(HERE, "sparse_traces.json"), "w") as f:
        json.dump(res, f)


def start_traces():
    """solve() with no start in feasible mode: phase 1 + shifted dual + centering
    (ipm_core.py:814-969) on the reference's random_feasible_lp instance."""
    from paper_2209_08722_b200.problems import random_feasible_dense
    A, b, c = random_feasible_dense(20, 200, 0.5, 3)
    ref_lp = skipm.random_feasible_lp(20, 200, 0.5, 3)
    assert np.array_equal(ref_lp.A.toarray(), A) and np.array_equal(ref_lp.b, b)
    res = {}
    prm = ipm_core.IpmParams(mode="feasible", gamma=0.5, sigma=0.5, tol_outer=1e-6, seed=2)
    x0, aux = ipm_core.phase1_point(ref_lp, prm)
    res["phase1_x0"] = x0.tolist()
    res["phase1_aux_outer"] = aux.outer
    st = ipm_core.feasible_start(ref_lp, prm)
    res["start"] = dict(x=st.x.tolist(), y=st.y.tolist(), s=st.s.tolist(), mu=st.mu)
    rep = ipm_core.solve(ref_lp, None, prm)
    d = rep.to_dict()
    d.pop("params")
    res["solve"] = d
    print(f"feasible start: aux outer {aux.outer}, start mu {st.mu:.4e}, solve outer {rep.outer} "
          f"obj {rep.objective!r}")
    with open(os.path.join(HERE, "start_traces.json"), "w") as f:
        json.dump(res, f)


def start_sparse_traces():
    """solve() with no start in feasible mode on a SPARSE LP (random_feasible_lp
    at 2% fill: CSC on the device, ~30% empty columns -> the zero-column fill),
    phase 1 and centering included (ipm_core.py:814-969)."""
    res = {}
    lp = skipm.random_feasible_lp(60, 4000, 0.02, 5)
    prm = ipm_core.IpmParams(mode="feasible", gamma=0.5, sigma=0.5, tol_outer=1e-6, seed=4)
    x0, aux = ipm_core.phase1_point(lp, prm)
    res["phase1_x0"] = x0.tolist()
    res["phase1_aux_outer"] = aux.outer
    st = ipm_core.feasible_start(lp, prm)
    res["start"] = dict(x=st.x.tolist(), y=st.y.tolist(), s=st.s.tolist(), mu=st.mu)
    rep = ipm_core.solve(lp, None, prm)
    d = rep.to_dict()
    d.pop("params")
    res["solve"] = d
    res["lp"] = dict(m=60, n=4000, density=0.02, seed=5, nnz=int(lp.A.nnz),
                     empty_cols=int((np.diff(lp.A.tocsc().indptr) == 0).sum()))
    print(f"sparse feasible start: aux outer {aux.outer}, start mu {st.mu:.4e}, solve outer "
          f"{rep.outer} obj {rep.objective!r}, empty cols {res['lp']['empty_cols']}")
    with open(os.path.join(HERE, "start_sparse_traces.json"), "w") as f:
        json.dump(res, f)


def write_libsvm_sample(path):
    """A small synthetic LIBSVM file (seeded; comments, blank lines, a repeated
    index, unsorted indices) for the ingestion parity test."""
    g = np.random.Generator(np.random.Philox(61))
    m, n = 30, 12
    X = np.where(g.random((m, n)) < 0.4, np.round(g.standard_normal((m, n)), 6), 0.0)
    y = np.sign(X @ g.standard_normal(n) + 1e-3)
    y[y == 0] = 1.0
    lines = ["# synthetic sample for tests/test_ingest.py", ""]
    for i in range(m):
        idx = [j for j in range(n) if X[i, j] != 0.0]
        g.shuffle(idx)
        toks = [f"{j + 1}:{float(X[i, j])!r}" for j in idx]
        if i == 3 and idx:
            toks.insert(0, f"{idx[0] + 1}:0.5")   # overwritten by the later token
        lines.append(f"{int(y[i]):+d} " + " ".join(toks) + ("  # row comment" if i == 5 else ""))
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def svm_traces():
    """Ingestion (load_libsvm, svm_to_lp) and the SVM pipeline solves of the
    reference's acceptance criterion 8 (test_acceptance.py:279-301)."""
    from skipm import lp_model
    path = os.path.join(HERE, "svm_small.libsvm")
    write_libsvm_sample(path)
    ds = lp_model.load_libsvm(path)
    lp, mp = lp_model.svm_to_lp(ds)
    np.savez(os.path.join(HERE, "svm_ingest.npz"), X=ds.X, y=ds.y, A_data=lp.A.data,
             A_indices=lp.A.indices, A_indptr=lp.A.indptr, b=lp.b, c=lp.c,
             shape=np.array(lp.A.shape))
    res = {}
    g = np.random.Generator(np.random.Philox(42))
    X50 = g.standard_normal((50, 100))
    y50 = np.sign(X50 @ g.standard_normal(100))
    cases = {"two_point": lp_model.SvmDataset(X=np.array([[1.0], [-1.0]]), y=np.array([1.0, -1.0])),
             "sep50x100": lp_model.SvmDataset(X=X50, y=y50), "libsvm_small": ds}
    for name, d in cases.items():
        lpc, mpc = lp_model.svm_to_lp(d)
        rep = ipm_core.solve(lpc, params=ipm_core.IpmParams(seed=0))
        w, b = lp_model.extract_svm_solution(mpc, rep.x)
        dd = rep.to_dict()
        dd.pop("params")
        res[name] = dict(outer=rep.outer, objective=rep.objective, converged=rep.converged,
                         mu_trace=list(map(float, rep.mu_trace)), w=w.tolist(), b=b,
                         w_l1=float(np.abs(w).sum()),
                         min_margin=float((d.y * (d.X @ w + b)).min()),
                         inner_iterations=[r.inner_iterations for r in rep.steps])
        print(f"svm {name}: outer {rep.outer} obj {rep.objective!r} converged {rep.converged}")
    with open(os.path.join(HERE, "svm_traces.json"), "w") as f:
        json.dump(res, f)


def diag_traces():
    """diag_cond=True (ipm_core.py:576-584): per-step spectrum bounds of the
    preconditioned normal matrix and cond(AD)^2 on a small LP."""
    lpd = wide_dense_lp(40, 3000, 5)
    A = lp_csr(lpd)
    st = ipm_core.make_iterate(skipm.make_lp(A, lpd.b, lpd.c), lpd.x0, lpd.y0, lpd.s0)
    prm = ipm_core.IpmParams(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=160, s=4,
                             tol_outer=1e-6, seed=3, diag_cond=True)
    rep = ipm_core.solve(skipm.make_lp(A, lpd.b, lpd.c), st, prm)
    res = {"outer": rep.outer,
           "steps": [{k: getattr(r, k) for k in ("spectrum_lo", "spectrum_hi", "kappa_sk",
                                                 "kappa_stan")} for r in rep.steps]}
    print(f"diag: outer {rep.outer}, kappa_sk max {max(r.kappa_sk for r in rep.steps):.3f}")
    with open(os.path.join(HERE, "diag_traces.json"), "w") as f:
        json.dump(res, f)


def lp_csr(lpd):
    import scipy.sparse as sp
    A = sp.csr_matrix(lpd.A)
    A.sort_indices()
    return A


if __name__ == "__main__":
    what = sys.argv[1:] or ["hashes", "adw", "small", "c1", "solvers", "start", "gaussian",
                            "sparse", "svm", "diag", "start_sparse"]
    if "svm" in what:
        svm_traces()
    if "diag" in what:
        diag_traces()
    if "sparse" in what:
        sparse_traces()
    if "gaussian" in what:
        gaussian_traces()
    if "start" in what:
        start_traces()
    if "start_sparse" in what:
        start_sparse_traces()
    if "solvers" in what:
        solver_traces()
    if "hashes" in what:
        hashes()
    if "adw" in what:
        adw()
    if "small" in what:
        small_traces()
    if "c1" in what:
        c1_traces()
