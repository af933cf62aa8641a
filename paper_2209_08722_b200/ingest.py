"""Problem ingestion: files and SVM data -> LP -> HBM.

Same entry points and error behaviour as the reference's loaders so a caller
can swap modules:

  load_libsvm(path) -> SvmDataset             reference lp_model.py:300-338
  svm_to_lp(ds) -> (LinearProgram, mapping)   reference lp_model.py:163-193
  extract_svm_solution(mapping, x)            reference lp_model.py:196-203
  save_matrix_market / load_matrix_market     reference lp_model.py:242-289
  to_device(lp)                               -> DeviceLP (CSC or column-major)

The LP is assembled straight into CSC triplets (the device layout of
sparse inputs, kernels.SparseDeviceMatrix) rather than by stacking CSR
blocks; `make_lp` then canonicalises to the reference's sorted CSR, so A is
identical entry for entry (the +-y x products are exact).
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np
import scipy.io
import scipy.sparse as sp

from .errors import DimensionMismatch, EmptyDataset, ParseError
from .lp_model import LinearProgram, make_lp


@dataclass
class SvmDataset:
    """Binary classification data: X is m x n, y in {-1, +1}^m."""

    X: np.ndarray
    y: np.ndarray


@dataclass
class SvmLpMapping:
    """Variable layout of svm_to_lp: [w+ (n), w- (n), b+, b-, xi (m)]."""

    n_features: int
    m_samples: int

    @property
    def n_lp(self) -> int:
        return 2 * self.n_features + 2 + self.m_samples


def svm_to_lp(ds: SvmDataset):
    """Hard-margin l1-SVM as a standard-form LP (reference lp_model.py:163-193):

        min 1'(w+ + w-)  s.t.  y_i x_i'(w+ - w-) + y_i (b+ - b-) - xi_i = 1,  all vars >= 0.
    """
    X = np.asarray(ds.X, dtype=np.float64)
    y = np.asarray(ds.y, dtype=np.float64)
    if X.ndim != 2 or 0 in X.shape:
        raise EmptyDataset(f"X has shape {X.shape}")
    m, n = X.shape
    if y.shape != (m,):
        raise DimensionMismatch(f"y has shape {y.shape}, expected ({m},)")
    if not np.all(np.abs(y) == 1.0):
        raise ParseError("labels must be -1 or +1")
    YX = sp.csc_matrix(y[:, None] * X)
    YX.eliminate_zeros()
    rows = np.arange(m)
    # column blocks in CSC: [YX | -YX | y | -y | -I]
    data = np.concatenate([YX.data, -YX.data, y, -y, -np.ones(m)])
    indices = np.concatenate([YX.indices, YX.indices, rows, rows, rows])
    nnz = YX.nnz
    colptr = np.concatenate([YX.indptr, nnz + YX.indptr[1:],
                             2 * nnz + m * np.arange(1, 3),
                             2 * nnz + 2 * m + np.arange(1, m + 1)])
    A = sp.csc_matrix((data, indices, colptr), shape=(m, 2 * n + 2 + m))
    b = np.ones(m)
    c = np.zeros(2 * n + 2 + m)
    c[:2 * n] = 1.0
    return make_lp(A, b, c, name=f"svm_{m}x{n}"), SvmLpMapping(n_features=n, m_samples=m)


def extract_svm_solution(mapping: SvmLpMapping, x) -> tuple[np.ndarray, float]:
    """(w, b) from an LP solution laid out per SvmLpMapping."""
    x = np.asarray(x)
    if x.shape != (mapping.n_lp,):
        raise DimensionMismatch(f"x has shape {x.shape}, expected ({mapping.n_lp},)")
    n = mapping.n_features
    return x[:n] - x[n:2 * n], float(x[2 * n] - x[2 * n + 1])


def load_libsvm(path: str) -> SvmDataset:
    """LIBSVM lines "label idx:val ..." (1-based indices, '#' comments), labels
    +-1; the feature count is the largest index seen."""
    labels, ri, ci, vals = [], [], [], []
    n = 0
    with open(path) as fh:
        for lineno, raw in enumerate(fh, 1):
            body = raw.partition("#")[0].split()
            if not body:
                continue
            try:
                lab = float(body[0])
            except ValueError as exc:
                raise ParseError(f"{path}:{lineno}: bad label {body[0]!r}") from exc
            if lab != 1.0 and lab != -1.0:
                raise ParseError(f"{path}:{lineno}: label must be -1 or +1, got {lab}")
            row = len(labels)
            seen = {}
            for tok in body[1:]:
                key, sep, val = tok.partition(":")
                try:
                    if not sep:
                        raise ValueError(tok)
                    j, v = int(key), float(val)
                except ValueError as exc:
                    raise ParseError(f"{path}:{lineno}: bad feature {tok!r}") from exc
                if j < 1:
                    raise ParseError(f"{path}:{lineno}: index {j} not 1-based")
                seen[j - 1] = v          # a repeated index keeps its last value
                n = max(n, j)
            labels.append(lab)
            ri.extend([row] * len(seen))
            ci.extend(seen.keys())
            vals.extend(seen.values())
    if not labels or n == 0:
        raise EmptyDataset(f"{path} holds no samples with features")
    X = np.zeros((len(labels), n))
    X[np.asarray(ri, dtype=np.int64), np.asarray(ci, dtype=np.int64)] = vals
    return SvmDataset(X=X, y=np.array(labels))


def save_matrix_market(lp: LinearProgram, directory: str) -> str:
    """A.mtx (17 significant digits), b.txt, c.txt and a problem.json manifest;
    values round-trip bit-identically through load_matrix_market."""
    os.makedirs(directory, exist_ok=True)
    scipy.io.mmwrite(os.path.join(directory, "A.mtx"), sp.csr_matrix(lp.A), precision=17)
    for stem, vec in (("b", lp.b), ("c", lp.c)):
        with open(os.path.join(directory, f"{stem}.txt"), "w") as fh:
            fh.writelines(f"{float(v)!r}\n" for v in vec)
    manifest = {"name": lp.name, "A": "A.mtx", "b": "b.txt", "c": "c.txt", "m": lp.m, "n": lp.n}
    path = os.path.join(directory, "problem.json")
    with open(path, "w") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return path


def _read_vector(path: str) -> np.ndarray:
    with open(path) as fh:
        toks = [t for t in (ln.strip() for ln in fh) if t]
    try:
        return np.array([float(t) for t in toks])
    except ValueError as exc:
        raise ParseError(f"bad vector file {path}: {exc}") from exc


def load_matrix_market(path: str) -> LinearProgram:
    """Problem from a problem.json manifest (or the directory holding one)."""
    if os.path.isdir(path):
        path = os.path.join(path, "problem.json")
    with open(path) as fh:
        try:
            manifest = json.load(fh)
        except json.JSONDecodeError as exc:
            raise ParseError(f"bad manifest {path}: {exc}") from exc
    base = os.path.dirname(path)
    try:
        A = scipy.io.mmread(os.path.join(base, manifest["A"]))
        b = _read_vector(os.path.join(base, manifest["b"]))
        c = _read_vector(os.path.join(base, manifest["c"]))
    except KeyError as exc:
        raise ParseError(f"manifest {path} missing key {exc}") from exc
    except ValueError as exc:
        raise ParseError(f"bad matrix file referenced by {path}: {exc}") from exc
    return make_lp(A, b, c, name=manifest.get("name", "lp"))


def to_device(lp: LinearProgram, comm=None, device=None):
    """Upload to HBM: CSC for sparse A (fill < lp_model.SPARSE_DENSITY), column-major
    otherwise; with a Comm, this rank's column block only."""
    from .lp_model import DeviceLP
    return DeviceLP.from_host(lp, comm=comm, device=device)
