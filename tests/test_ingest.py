"""Problem ingestion (LIBSVM, SVM LP, Matrix Market) against the reference's
outputs (tests/golden/make_golden.py svm) and its own test cases
(reference tests/test_lp_model.py:127-200, test_acceptance.py:279-301)."""

import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN
from paper_2209_08722_b200 import ingest as I
from paper_2209_08722_b200.errors import DimensionMismatch, EmptyDataset, ParseError
from paper_2209_08722_b200.lp_model import make_lp


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "svm_ingest.npz"))


def test_libsvm_and_svm_lp_match_reference(gold):
    ds = I.load_libsvm(os.path.join(GOLDEN, "svm_small.libsvm"))
    assert np.array_equal(ds.X, gold["X"]) and np.array_equal(ds.y, gold["y"])
    lp, mp = I.svm_to_lp(ds)
    assert lp.A.shape == tuple(gold["shape"])
    assert np.array_equal(lp.A.indptr, gold["A_indptr"])
    assert np.array_equal(lp.A.indices, gold["A_indices"])
    assert np.array_equal(lp.A.data, gold["A_data"])
    assert np.array_equal(lp.b, gold["b"]) and np.array_equal(lp.c, gold["c"])
    assert mp.n_lp == lp.n == 2 * ds.X.shape[1] + 2 + ds.X.shape[0]


def test_two_point_shape_and_costs():
    lp, mp = I.svm_to_lp(I.SvmDataset(X=np.array([[1.0], [-1.0]]), y=np.array([1.0, -1.0])))
    assert (lp.m, lp.n) == (2, 6) and mp.n_lp == 6
    lp, _ = I.svm_to_lp(I.SvmDataset(X=np.ones((3, 4)), y=np.array([1.0, -1.0, 1.0])))
    assert np.all(lp.c >= 0) and int(np.sum(lp.c == 1.0)) == 8
    assert int(np.sum(lp.c == 0.0)) == lp.n - 8


@pytest.mark.parametrize("X,y,exc", [
    (np.zeros((0, 3)), np.zeros(0), EmptyDataset),
    (np.ones((2, 2)), np.array([1.0, 2.0]), ParseError),
    (np.ones((2, 2)), np.array([1.0, -1.0, 1.0]), DimensionMismatch),
])
def test_svm_to_lp_errors(X, y, exc):
    with pytest.raises(exc):
        I.svm_to_lp(I.SvmDataset(X=X, y=y))


def test_margin_residual_identity():
    """Any point with Ax = b reproduces y_i (w'x_i + b) - 1 = xi_i."""
    for seed in range(12):
        g = np.random.Generator(np.random.Philox(seed))
        m, n = 1 + seed % 6, 1 + seed % 5
        X = g.standard_normal((m, n))
        y = np.where(g.random(m) < 0.5, 1.0, -1.0)
        lp, mp = I.svm_to_lp(I.SvmDataset(X=X, y=y))
        free = g.random(lp.n) + 0.1
        x = free + np.linalg.lstsq(lp.A.toarray(), lp.b - lp.A @ free, rcond=None)[0]
        w, b = I.extract_svm_solution(mp, x)
        xi = x[2 * n + 2:]
        assert np.max(np.abs(y * (X @ w + b) - 1.0 - xi)) <= 1e-12 * max(1.0, np.abs(xi).max())


def test_extract_svm_solution():
    mp = I.SvmLpMapping(n_features=2, m_samples=1)
    w, b = I.extract_svm_solution(mp, np.array([0.5, 0.5, 0.5, 0.5, 0.25, 0.25, 0.0]))
    assert np.array_equal(w, [0.0, 0.0]) and b == 0.0
    with pytest.raises(DimensionMismatch):
        I.extract_svm_solution(mp, np.zeros(5))


@pytest.mark.parametrize("body,exc", [
    ("2 1:1.0\n", ParseError), ("+1 1:abc\n", ParseError), ("+1 0:1.0\n", ParseError),
    ("x 1:1\n", ParseError), ("+1 1\n", ParseError), ("# only a comment\n\n", EmptyDataset),
    ("+1\n-1\n", EmptyDataset),
])
def test_libsvm_parse_errors(tmp_path, body, exc):
    p = tmp_path / "d.libsvm"
    p.write_text(body)
    with pytest.raises(exc):
        I.load_libsvm(str(p))


def test_matrix_market_round_trip_bit_identical(tmp_path):
    g = np.random.Generator(np.random.Philox(13))
    A = np.where(g.random((6, 18)) < 0.5, g.standard_normal((6, 18)) / 3.0, 0.0)
    A[np.arange(6), np.arange(6)] += 1.0
    lp = make_lp(A, g.standard_normal(6) / 7.0, g.random(18) * np.pi, name="rt")
    manifest = I.save_matrix_market(lp, str(tmp_path / "prob"))
    back = I.load_matrix_market(os.path.dirname(manifest))
    assert back.name == "rt"
    assert np.array_equal(back.A.toarray(), lp.A.toarray())
    assert np.array_equal(back.b, lp.b) and np.array_equal(back.c, lp.c)
    with open(manifest) as f:
        assert json.load(f)["n"] == 18


def test_matrix_market_errors(tmp_path):
    d = tmp_path / "bad"
    d.mkdir()
    (d / "problem.json").write_text("{not json")
    with pytest.raises(ParseError):
        I.load_matrix_market(str(d))
    (d / "problem.json").write_text(json.dumps({"A": "A.mtx"}))
    with pytest.raises((ParseError, FileNotFoundError)):
        I.load_matrix_market(str(d))


# ------------------------------------------------------- SVM pipeline (GPU)
def _cases():
    g = np.random.Generator(np.random.Philox(42))
    X = g.standard_normal((50, 100))
    y = np.sign(X @ g.standard_normal(100))
    return {"two_point": I.SvmDataset(X=np.array([[1.0], [-1.0]]), y=np.array([1.0, -1.0])),
            "sep50x100": I.SvmDataset(X=X, y=y),
            "libsvm_small": I.load_libsvm(os.path.join(GOLDEN, "svm_small.libsvm"))}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["two_point", "sep50x100", "libsvm_small"])
def test_svm_pipeline_matches_reference(name):
    """solve(lp, params=IpmParams(seed=0)) with no start (phase 1 + centering on
    the device) on the reference's acceptance-criterion-8 problems."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_08722_b200 import ipm_core as IC
    with open(os.path.join(GOLDEN, "svm_traces.json")) as f:
        gold = json.load(f)[name]
    ds = _cases()[name]
    lp, mp = I.svm_to_lp(ds)
    rep = IC.solve(lp, params=IC.IpmParams(seed=0))
    w, b = I.extract_svm_solution(mp, rep.x)
    assert rep.converged
    assert rep.outer == gold["outer"]
    assert abs(rep.objective - gold["objective"]) <= 1e-8 * abs(gold["objective"])
    assert float((ds.y * (ds.X @ w + b)).min()) >= 1.0 - 1e-6
    if name == "two_point":
        assert abs(float(np.abs(w).sum()) - 1.0) <= 1e-6


def test_null_pair_columns():
    """Zero-cost anti-parallel pairs (reference ipm_core.py:737-760): each column
    matched at most once, in column order; nonzero-cost columns never pair."""
    from paper_2209_08722_b200.ipm_core import _null_pair_columns
    from paper_2209_08722_b200.lp_model import LinearProgram
    lp, mp = I.svm_to_lp(I.SvmDataset(X=np.array([[1.0, 2.0], [-1.0, 0.5]]),
                                      y=np.array([1.0, -1.0])))
    assert _null_pair_columns(lp) == [(4, 5)]          # b+ / b-; w+/w- cost 1
    a = np.array([1.0, -2.0, 0.0])
    A = np.stack([a, -a, -a, a, a, 2 * a, np.array([0.0, 0.0, 1.0])], axis=1)
    c = np.array([0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0])
    assert _null_pair_columns(LinearProgram(sp.csr_matrix(A), np.ones(3), c)) == [(0, 1), (2, 3)]


def test_reference_generators_identical():
    """random_lp / random_feasible_lp reproduce the reference's instances
    (tests/golden/start_traces.json pins random_feasible_lp(20, 200, 0.5, 3))."""
    from paper_2209_08722_b200 import random_feasible_lp, random_lp
    from paper_2209_08722_b200.errors import DimensionMismatch, InvalidDensity
    lp = random_feasible_lp(20, 200, 0.5, 3)
    assert lp.name == "random_feasible_lp_20x200_d0.5_s3" and lp.A.shape == (20, 200)
    with open(os.path.join(GOLDEN, "start_traces.json")) as f:
        gold = json.load(f)
    x0 = np.array(gold["phase1_x0"])            # A x0 = b for the reference's instance
    assert np.linalg.norm(lp.A @ x0 - lp.b) <= 1e-6 * np.linalg.norm(lp.b)
    with pytest.raises(InvalidDensity):
        random_lp(3, 5, 0.0, 1)
    with pytest.raises(DimensionMismatch):
        random_lp(5, 3, 0.5, 1)
    assert random_lp(4, 9, 0.5, 2).name == "random_lp_4x9_d0.5_s2"
