"""CPU-side checks: the C-ABI library loads and exports every symbol that
include/skb.h declares, the header binding is well formed, and the host
helpers (sketch dims, t_max, sharding) match the reference's formulas."""

import ctypes
import math
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2209_08722_b200", "libskb.so")


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        from paper_2209_08722_b200 import build
        build.build()
    return LIB


def test_header_parses_and_every_symbol_is_exported(built):
    from paper_2209_08722_b200 import _lib
    protos = _lib.parse_header()
    assert len(protos) >= 35
    nm = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True,
                        check=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if " T " in line}
    missing = sorted(set(protos) - exported)
    assert not missing, missing
    L = ctypes.CDLL(built)  # loads without a GPU (no compute calls here)
    for name in protos:
        assert hasattr(L, name)


def test_sass_contains_dmma_and_bulk_copies(built):
    sass = subprocess.run(["cuobjdump", "-sass", built], capture_output=True, text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "DMMA" in sass          # FP64 tensor-core GEMM (mma.sync f64)
    assert "UBLKCP" in sass        # cp.async.bulk (TMA bulk engine) in the streaming kernels


def test_auto_sketch_dims_and_t_max_reference_values():
    from paper_2209_08722_b200.ipm_core import IpmParams, default_t_max
    from paper_2209_08722_b200.sketching import auto_sketch_dims
    # tests/test_sketching.py:236-239 and tests/test_ipm_core.py:407-410 of the reference
    assert auto_sketch_dims(20, 2000, 5e-4) == (2000, 16)
    assert auto_sketch_dims(20, 4000, 5e-4) == (2560, 16)
    assert default_t_max(400, IpmParams()) == 15
    p = IpmParams(gamma=0.749, sigma=0.5, zeta=0.5)
    assert [default_t_max(n, p) for n in (10_000, 1_000_000, 4_000_000, 20_000_000)] == \
        [19, 26, 28, 30]


def test_params_validation_matches_reference():
    from paper_2209_08722_b200.errors import InvalidZeta
    from paper_2209_08722_b200.ipm_core import IpmParams
    IpmParams().validate()
    for kw in (dict(gamma=0.0), dict(sigma=0.8), dict(mode="x"), dict(max_outer=0),
               dict(sketch="y"), dict(tol_cg=0.0)):
        with pytest.raises(ValueError):
            IpmParams(**kw).validate()
    with pytest.raises(InvalidZeta):
        IpmParams(zeta=1.0).validate()
    assert IpmParams(max_outer=200).delta == 0.1 / 200


def test_shard_ranges_cover_columns():
    from paper_2209_08722_b200.distributed import shard_range
    for n in (1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(j1 - j0 for j0, j1 in rs) - min(j1 - j0 for j0, j1 in rs) <= 1


def test_host_validate_matches_reference_rules():
    import scipy.sparse as sp
    from paper_2209_08722_b200.errors import DimensionMismatch, ZeroRow
    from paper_2209_08722_b200.lp_model import LinearProgram, make_lp, validate
    make_lp(np.eye(2, 3) + 0.1, np.ones(2), np.ones(3))
    with pytest.raises(DimensionMismatch):
        make_lp(np.ones((3, 2)), np.ones(3), np.ones(2))
    A = np.ones((2, 3))
    A[1] = 0.0
    with pytest.raises(ZeroRow):
        validate(LinearProgram(sp.csr_matrix(A), np.ones(2), np.ones(3)))


def test_first_crossing_scalar_matches_oracle():
    from oracle import ipm_oracle as O
    from paper_2209_08722_b200.ipm_core import _first_crossing_scalar
    rng = np.random.default_rng(0)
    for _ in range(500):
        a, b, c = rng.standard_normal(3) * 10.0 ** rng.uniform(-3, 3, 3)
        if rng.random() < 0.2:
            a = 0.0
        if rng.random() < 0.1:
            c = -abs(c) * 1e-14
        ref = O.first_crossing(np.array([a]), np.array([b]), np.array([c]))
        got = _first_crossing_scalar(a, b, c)
        assert (ref == got) or (math.isinf(ref) and math.isinf(got))


def test_first_crossing_scalar_bitwise_equals_numpy_form():
    """The plain-float _first_crossing_scalar (the step's host path) against the
    reference's numpy expression restated for one quadratic: bitwise equal on
    special values (+-0, +-inf, NaN, subnormals, 1e+-300) and 1e5 random cases
    spanning 40 decades, incl. a = 0 and c slightly negative."""
    import itertools
    import math
    import warnings
    from paper_2209_08722_b200.ipm_core import _first_crossing_np, _first_crossing_scalar
    sp_ = [0.0, -0.0, 1e-300, -1e-300, 1e300, -1e300, math.inf, -math.inf, math.nan, 1.0, -1.0,
           1e-12, -1e-13, 5e-324]
    g = np.random.Generator(np.random.Philox(17))
    cases = list(itertools.product(sp_, repeat=3))
    for _ in range(100_000):
        a, b, c = g.standard_normal(3) * 10.0 ** g.uniform(-20, 20, 3)
        if g.random() < 0.2:
            a = 0.0
        if g.random() < 0.1:
            c = -abs(c) * 1e-14
        cases.append((a, b, c))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for a, b, c in cases:
            x, y = _first_crossing_scalar(a, b, c), _first_crossing_np(a, b, c)
            assert (x == y and math.copysign(1, x) == math.copysign(1, y)) or \
                (math.isnan(x) and math.isnan(y)), (a, b, c, x, y)
