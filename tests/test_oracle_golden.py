"""Pin the oracle (oracle/) against fixtures produced by the live reference
(tests/golden/make_golden.py). CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import chash
from oracle import ipm_oracle as O
from paper_2209_08722_b200.problems import wide_dense_lp

from conftest import GOLDEN


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def hashes():
    return np.load(os.path.join(GOLDEN, "hashes.npz"))


@pytest.fixture(scope="module")
def big():
    with open(os.path.join(GOLDEN, "hashes_big.json")) as f:
        return json.load(f)


def _cases(h):
    for k in h.files:
        if k.startswith("cols_"):
            n, w, s, seed = map(int, k[5:].split("_"))
            yield n, w, s, seed, h[k], h["sign_" + k[5:]]


def test_numpy_restatement_matches_reference_hashes(hashes):
    for n, w, s, seed, cols, sign in _cases(hashes):
        c, v = O.sparse_embedding(n, w, s, seed)
        assert np.array_equal(c, cols), (n, w, s, seed)
        assert np.array_equal(v > 0, sign.astype(bool))
        assert np.all(np.abs(v) == 1.0 / np.sqrt(s))


def test_c_restatement_matches_reference_hashes(hashes):
    checked = 0
    for n, w, s, seed, cols, sign in _cases(hashes):
        if 2 * s >= w:
            continue
        c, v, used = chash.sparse_embedding(n, w, s, seed)
        assert np.array_equal(c, cols), (n, w, s, seed)
        assert np.array_equal(v > 0, sign.astype(bool))
        checked += 1
    assert checked >= 7


def test_c_lemire_matches_numpy_with_rejections(hashes):
    for w in (3 * 2**30, 2**31 + 1, 5):
        out, used = chash.lemire_draw(21, w, 4000)
        assert np.array_equal(out, hashes[f"lemire_{w}"])
        if w == 3 * 2**30:
            assert used > 4000 + 500   # threshold 2^30: ~25% of words rejected


def test_c_big_hash_checksums(big):
    for case in big["big"]:
        if case["s"] * case["n"] > 4_000_000:
            continue
        c, v, _ = chash.sparse_embedding(case["n"], case["w"], case["s"], case["seed"])
        assert _sha(c) == case["cols_sha256"]
        assert _sha((v > 0).astype(np.int8)) == case["sign_sha256"]


def test_outer_seed_stream(big):
    for seed, rec in big["outer_seeds"].items():
        assert list(chash.philox_key(int(seed))) == rec["key"]
        assert [chash.out64(int(seed), k) >> 1 for k in range(8)] == rec["draws"]


def test_adw_bits():
    g = np.load(os.path.join(GOLDEN, "adw_small.npz"))
    A, d = g["A"], g["d"]
    Acsr = sp.csr_matrix(A)
    for s in (1, 4):
        cols, vals = O.sparse_embedding(A.shape[1], 64, s, int(g[f"seed_s{s}"]))
        ref = g[f"adw_s{s}"]
        assert np.array_equal(chash.adw_dense(A, d, cols, vals, 64), ref)
        W = O.Sketch("sparse_sign", A.shape[1], 64, s, 0, cols=cols, vals=vals)
        assert np.array_equal(O.apply_sketch(Acsr, d, W), ref)


def test_normal_op_pcg_factor():
    g = np.load(os.path.join(GOLDEN, "adw_small.npz"))
    A, d, v = sp.csr_matrix(g["A"]), g["d"], g["v"]
    op = O.NormalOp(A, d)
    np.testing.assert_allclose(op.apply(v), g["normal_apply"], rtol=1e-13, atol=0)
    cols, vals = O.sparse_embedding(A.shape[1], 64, 4, 104)
    W = O.Sketch("sparse_sign", A.shape[1], 64, 4, 104, cols=cols, vals=vals)
    f = O.Factor(O.apply_sketch(A, d, W))
    np.testing.assert_allclose(f.inv(v), g["inv_v"], rtol=1e-11)
    np.testing.assert_allclose(f.pinv(v), g["pinv_v"], rtol=1e-11)
    dy, norms, its, conv = O.pcg(op, f, v, 30, 1e-10)
    np.testing.assert_allclose(dy, g["pcg_dy"], rtol=1e-10)
    np.testing.assert_allclose(norms, g["pcg_norms"], rtol=1e-8)


def _oracle_problem(m, n, seed):
    lpd = wide_dense_lp(m, n, seed)
    A = sp.csr_matrix(lpd.A)
    A.sort_indices()
    return lpd, A


def _compare_solve(rep, gold, mu_rtol):
    assert rep["outer"] == gold["outer"]
    assert [r["inner_iterations"] for r in rep["steps"]] == gold["inner_iterations"]
    assert [r["sketch_seed"] for r in rep["steps"]] == [s["sketch_seed"] for s in gold["steps"]]
    np.testing.assert_allclose(rep["mu_trace"], gold["mu_trace"], rtol=mu_rtol)
    assert abs(rep["objective"] - gold["objective"]) <= 1e-10 * abs(gold["objective"])


def test_small_traces_both_modes():
    with open(os.path.join(GOLDEN, "small_traces.json")) as f:
        gold = json.load(f)
    lpd, A = _oracle_problem(40, 3000, 5)
    st = O.make_iterate(A, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0)
    prm = O.Params(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=160, s=4,
                   tol_outer=1e-7, seed=3)
    _compare_solve(O.solve(A, lpd.b, lpd.c, st, prm), gold["feasible"], 1e-12)
    st = O.make_iterate(A, lpd.b, lpd.c, np.ones(3000), np.zeros(40), np.ones(3000))
    prm = O.Params(mode="infeasible", gamma=0.5, sigma=0.5, w=160, s=4, tol_outer=1e-7,
                   seed=4, max_outer=60)
    _compare_solve(O.solve(A, lpd.b, lpd.c, st, prm), gold["infeasible"], 1e-12)


@pytest.mark.parametrize("s_nnz", [4, 1])
def test_config1_trace(s_nnz):
    with open(os.path.join(GOLDEN, "c1_traces.json")) as f:
        gold = json.load(f)
    lpd, A = _oracle_problem(100, 10_000, 0)
    st = O.make_iterate(A, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0)
    prm = O.Params(mode="feasible", gamma=gold["gamma_run"], sigma=0.5, w=400, s=s_nnz,
                   tol_outer=1e-6, seed=0)
    _compare_solve(O.solve(A, lpd.b, lpd.c, st, prm), gold[f"s{s_nnz}"], 1e-12)


def test_sparse_config_trace_and_adw():
    from paper_2209_08722_b200.problems import sparse_wide_lp
    with open(os.path.join(GOLDEN, "sparse_traces.json")) as f:
        gold = json.load(f)
    lpd = sparse_wide_lp(100, 20_000, 5, 7)
    A = sp.csr_matrix(lpd.A)
    A.sort_indices()
    st = O.make_iterate(A, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0)
    prm = O.Params(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, w=400, s=4,
                   tol_outer=1e-6, seed=11)
    _compare_solve(O.solve(A, lpd.b, lpd.c, st, prm), gold["s4"], 1e-12)
    cols, vals = O.sparse_embedding(lpd.n, 400, 4, 77)
    d = 10.0 ** np.random.Generator(np.random.Philox(78)).uniform(-3, 3, lpd.n)
    W = O.Sketch("sparse_sign", lpd.n, 400, 4, 77, cols=cols, vals=vals)
    assert _sha(O.apply_sketch(A, d, W)) == gold["adw_sha256"]


def test_gaussian_sketch_and_traces():
    from paper_2209_08722_b200.problems import ill_conditioned_lp
    with open(os.path.join(GOLDEN, "gaussian_traces.json")) as f:
        gold = json.load(f)
    for case in gold["sketch"]:
        W = O.gaussian_sketch(case["n"], case["w"], case["seed"])
        assert _sha(W) == case["sha256"]
    for name, lpd in [("wide", wide_dense_lp(40, 3000, 5)), ("illcond", ill_conditioned_lp(30, 2000, 6))]:
        A = sp.csr_matrix(lpd.A)
        A.sort_indices()
        st = O.make_iterate(A, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0)
        prm = O.Params(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5 if name == "wide" else 0.3,
                       sketch="gaussian", w=4 * lpd.m, tol_outer=1e-6, seed=9)
        _compare_solve(O.solve(A, lpd.b, lpd.c, st, prm), gold[name], 1e-12)


@pytest.mark.parametrize("name", ["chebyshev", "unpreconditioned", "direct", "pcg_nocorr"])
def test_other_solvers_traces(name):
    with open(os.path.join(GOLDEN, "solver_traces.json")) as f:
        gold = json.load(f)[name]
    kw = {"chebyshev": dict(solver="chebyshev", w=1200, s=12),
          "unpreconditioned": dict(solver="unpreconditioned", w=160, s=4),
          "direct": dict(solver="direct", w=160, s=4),
          "pcg_nocorr": dict(solver="pcg", correction=False, w=160, s=4)}[name]
    lpd, A = _oracle_problem(40, 3000, 5)
    st = O.make_iterate(A, lpd.b, lpd.c, lpd.x0, lpd.y0, lpd.s0)
    prm = O.Params(mode="feasible", gamma=lpd.gamma_run(0.1), sigma=0.5, tol_outer=1e-6, seed=5,
                   **kw)
    rep = O.solve(A, lpd.b, lpd.c, st, prm)
    assert rep["outer"] == gold["outer"]
    assert [r["inner_iterations"] for r in rep["steps"]] == gold["inner_iterations"]
    np.testing.assert_allclose(rep["mu_trace"], gold["mu_trace"], rtol=1e-12)
    assert abs(rep["objective"] - gold["objective"]) <= 1e-10 * abs(gold["objective"])


def test_glibc_log1p_restatement_matches_host_libm(tmp_path):
    """The explicit-FMA log1p that csrc/skb_gauss.cu uses in the ziggurat tail
    (tests/golden/log1p_check.c, the same operations in C) equals the host
    libm's log1p -- numpy's npy_log1p -- bit for bit on 2e7 arguments in (-1, 0]."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no C compiler")
    exe = tmp_path / "log1p_check"
    src = os.path.join(os.path.dirname(__file__), "golden", "log1p_check.c")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", src, "-lm", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "20000000"], capture_output=True, text=True)
    print(out.stdout.strip())
    assert out.returncode == 0 and "mismatches 0" in out.stdout
