"""GPU parity of the individual kernels against the oracle / golden fixtures."""

import hashlib
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import GOLDEN
from oracle import chash
from oracle import ipm_oracle as O

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


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ----------------------------------------------------------------- hashes


def test_hash_tables_bit_exact(K):
    g = np.load(os.path.join(GOLDEN, "hashes.npz"))
    for key in g.files:
        if not key.startswith("cols_"):
            continue
        n, w, s, seed = map(int, key[5:].split("_"))
        k0, k1 = chash.philox_key(seed)
        cols, vals, used = K.sparse_embedding(k0, k1, n, w, s)
        assert np.array_equal(_h(cols).astype(np.int64), g[key]), (n, w, s, seed)
        assert np.array_equal(_h(vals) > 0, g["sign_" + key[5:]].astype(bool))
        assert np.all(np.abs(_h(vals)) == 1.0 / np.sqrt(s))


def test_hash_words_consumed_match_c_oracle(K):
    for (n, w, s, seed) in [(10_000, 400, 1, 11), (3_000, 400, 18, 14), (1_000, 40, 4, 17)]:
        k0, k1 = chash.philox_key(seed)
        _, _, used = K.sparse_embedding(k0, k1, n, w, s)
        _, _, used_c = chash.sparse_embedding(n, w, s, seed)
        assert used == used_c


def test_hash_full_size_checksums(K):
    with open(os.path.join(GOLDEN, "hashes_big.json")) as f:
        big = json.load(f)
    for case in big["big"]:
        k0, k1 = chash.philox_key(case["seed"])
        cols, vals, _ = K.sparse_embedding(k0, k1, case["n"], case["w"], case["s"])
        c = _h(cols).astype(np.int64)
        assert _sha(c) == case["cols_sha256"], case
        assert _sha((_h(vals) > 0).astype(np.int8)) == case["sign_sha256"]


def test_lemire_draws_with_rejections(K):
    g = np.load(os.path.join(GOLDEN, "hashes.npz"))
    for w in (3 * 2**30, 2**31 + 1, 5):
        k0, k1 = chash.philox_key(21)
        out, used = K.lemire_draw(k0, k1, w, 4000)
        assert np.array_equal(_h(out), g[f"lemire_{w}"])
        _, used_c = chash.lemire_draw(21, w, 4000)
        assert used == used_c


# ---------------------------------------------------------- column streams

# m > ~13,900 (and > 16,384): the two-pass global-memory fallback of the dense passes
SHAPES = [(1, 7), (20, 600), (63, 1000), (100, 10_000), (257, 3000), (1000, 5000),
          (1001, 4001), (1025, 3000), (2000, 3000), (3001, 2500), (5000, 1200),
          (16_000, 700), (20_001, 333)]


def _problem(m, n, seed=0):
    g = np.random.Generator(np.random.Philox(seed))
    A = g.standard_normal((m, n))
    return g, A


@pytest.mark.parametrize("m,n", SHAPES)
def test_normal_apply(K, m, n):
    g, A = _problem(m, n)
    d = 10.0 ** g.uniform(-2, 2, n)
    z = g.standard_normal(m)
    Ad = K.DeviceMatrix.from_host(A)
    d2 = d**2
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    K.normal_apply(Ad, _t(d2), _t(z), out)
    ref = O.NormalOp(sp.csr_matrix(A), d).apply(z)
    scale = np.abs(A).dot(d2 * np.abs(A.T @ z)).max() + 1e-300
    assert np.max(np.abs(_h(out) - ref)) <= 1e-13 * scale
    # deterministic run to run
    out2 = torch.empty_like(out)
    K.normal_apply(Ad, _t(d2), _t(z), out2, sub=_t(ref))
    assert np.array_equal(_h(out2), _h(out) - ref)


@pytest.mark.parametrize("m,n", SHAPES)
def test_gemv_and_transpose(K, m, n):
    g, A = _problem(m, n, 1)
    x, y, s, c = g.standard_normal(n), g.standard_normal(m), g.random(n) + 0.5, g.standard_normal(n)
    b = g.standard_normal(m)
    Ad = K.DeviceMatrix.from_host(A)
    u = torch.empty(m, dtype=torch.float64, device="cuda")
    K.gemv(Ad, _t(x), u, sub=_t(b))
    ref = A @ x - b
    assert np.max(np.abs(_h(u) - ref)) <= 1e-13 * (np.abs(A) @ np.abs(x)).max()
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    K.gemv_t(Ad, _t(y), t, add=_t(s), sub=_t(c))
    ref = A.T @ y + s - c
    assert np.max(np.abs(_h(t) - ref)) <= 1e-13 * (np.abs(A.T) @ np.abs(y) + 1).max()
    K.gemv_ratio(Ad, _t(x), _t(s), u)
    ref = A @ (x / s)
    assert np.max(np.abs(_h(u) - ref)) <= 1e-13 * (np.abs(A) @ np.abs(x / s)).max()


@pytest.mark.parametrize("mode", ["feasible", "infeasible"])
def test_rhs_directions_iterate(K, mode):
    m, n = 300, 4000
    g, A = _problem(m, n, 2)
    x, s = g.random(n) + 0.2, g.random(n) + 0.2
    y, dy = g.standard_normal(m), g.standard_normal(m)
    v = 1e-3 * g.standard_normal(n)
    r_d = 1e-2 * g.standard_normal(n) if mode == "infeasible" else None
    r_p = 1e-2 * g.standard_normal(m) if mode == "infeasible" else None
    b, c = g.standard_normal(m), g.standard_normal(n)
    smu = 0.5 * 0.37
    Acsr = sp.csr_matrix(A)
    Ad = K.DeviceMatrix.from_host(A)
    it = O.Iterate(x, y, s, r_p if r_p is not None else np.zeros(m),
                   r_d if r_d is not None else np.zeros(n), 0.37)
    p = torch.empty(m, dtype=torch.float64, device="cuda")
    K.rhs(Ad, _t(x), _t(s), smu, p, r_d=None if r_d is None else _t(r_d),
          r_p=None if r_p is None else _t(r_p))
    ref = O.build_rhs(Acsr, it, 0.5, mode)
    assert np.max(np.abs(_h(p) - ref)) <= 1e-12 * np.abs(ref).max()

    ds, dx, adx, atdy = (torch.empty(n, dtype=torch.float64, device="cuda"),
                         torch.empty(n, dtype=torch.float64, device="cuda"),
                         torch.empty(m, dtype=torch.float64, device="cuda"),
                         torch.empty(n, dtype=torch.float64, device="cuda"))
    K.directions(Ad, _t(dy), _t(x), _t(s), _t(v), smu, ds, dx, adx, atdy=atdy,
                 r_d=None if r_d is None else _t(r_d))
    Atdy = A.T @ dy
    ds_ref = -Atdy if mode == "feasible" else -r_d - Atdy
    dx_ref = -x + smu / s - (x / s) * ds_ref - v / s
    assert np.max(np.abs(_h(atdy) - Atdy)) <= 1e-13 * np.abs(Atdy).max()
    assert np.max(np.abs(_h(ds) - ds_ref)) <= 1e-13 * np.abs(ds_ref).max()
    assert np.max(np.abs(_h(dx) - dx_ref)) <= 1e-12 * np.abs(dx_ref).max()
    # elementwise formulas are bit-exact given the same A'dy
    ds_from = -_h(atdy) if mode == "feasible" else -r_d - _h(atdy)
    assert np.array_equal(_h(ds), ds_from)
    assert np.array_equal(_h(dx), -x + smu / s - (x / s) * ds_from - v / s)
    adx_ref = A @ _h(dx)
    assert np.max(np.abs(_h(adx) - adx_ref)) <= 1e-13 * (np.abs(A) @ np.abs(_h(dx))).max()

    alpha = 0.61
    xo, so = torch.empty_like(ds), torch.empty_like(ds)
    rp, rd = torch.empty_like(adx), torch.empty_like(ds)
    ynew = y + alpha * dy
    K.iterate(Ad, _t(x), _t(s), _t(ynew), _t(b), _t(c), rp, rd, dx=dx, ds=ds, alpha=alpha,
              x_out=xo, s_out=so)
    xn, sn = x + alpha * _h(dx), s + alpha * _h(ds)
    assert np.array_equal(_h(xo), xn) and np.array_equal(_h(so), sn)
    ref_rp, ref_rd = A @ xn - b, A.T @ ynew + sn - c
    assert np.max(np.abs(_h(rp) - ref_rp)) <= 1e-13 * (np.abs(A) @ np.abs(xn)).max()
    assert np.max(np.abs(_h(rd) - ref_rd)) <= 1e-13 * (np.abs(A.T) @ np.abs(ynew) + 1).max()


# ------------------------------------------------------------ DMMA GEMM
GEMM_CASES = [(129, 65, 37, 0), (300, 200, 1000, 0), (1000, 1000, 4000, 1), (64, 64, 16, 0),
              (257, 130, 3, 0), (1024, 512, 2048, 1)]


@pytest.mark.parametrize("M,N,Kd,lower", GEMM_CASES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("pipe", ["pipe", "nopipe", "emu"])
def test_gemm_against_numpy(K, monkeypatch, M, N, Kd, lower, ta, tb, pipe):
    """skb_gemm (the cp.async 128x64 DMMA kernel, the register-staged fallback,
    and the INT8 emulation forced for K >= 256) against numpy fp64; error bound
    1e-13 * sum|a||b|."""
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    monkeypatch.setenv("SKB_GEMM_EMU", "2" if pipe == "emu" else "0")
    if pipe == "nopipe":
        monkeypatch.setenv("SKB_GEMM_NOPIPE", "1")
    g = np.random.Generator(np.random.Philox(M * 7 + N + Kd))
    opa = g.standard_normal((M, Kd))
    opb = g.standard_normal((Kd, N))
    A = opa.T.copy() if ta else opa.copy()
    B = opb.T.copy() if tb else opb.copy()
    C0 = g.standard_normal((M, N))
    Cd = _t(C0)
    ws, cap = workspace((1 << 26) + int(_lib.lib().skb_gemm_ozaki_workspace_bytes(M, N, Kd)))
    _lib.call("skb_gemm", ta, tb, M, N, Kd, 0.5, _t(A), A.shape[1], _t(B), B.shape[1], -1.0, Cd, N,
              lower, 1, 0, 0, 0, ws, cap, stream_ptr())
    ref = 0.5 * opa @ opb - C0
    bound = 1e-13 * (np.abs(opa) @ np.abs(opb) + np.abs(C0))
    out = _h(Cd)
    mask = np.tril(np.ones((M, N), bool)) if lower else np.ones((M, N), bool)
    assert np.all(np.abs(out - ref)[mask] <= bound[mask])


def test_weighted_gram(K):
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(12))
    m, n = 300, 5000
    A = g.standard_normal((m, n))
    wts = g.random(n) + 0.1
    G = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    ws, cap = workspace(1 << 26)
    _lib.call("skb_weighted_gram", _t(A.T), m, n, m, _t(wts), G, m, ws, cap, stream_ptr())
    ref = (A * wts) @ A.T
    out = np.tril(_h(G))
    assert np.max(np.abs(out - np.tril(ref))) <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("Mp,emu", [(192, "0"), (1024, "0"), (2560, "0"), (1024, "2"),
                                    (2560, "2"), (4160, "1"), (8192, "1")])
def test_potrf_trtri_against_numpy(K, monkeypatch, Mp, emu):
    """skb_potrf (64-wide panels; two-level 512-wide blocking from Mp = 2048)
    and skb_trtri against numpy's Cholesky / inverse on an SPD Gram matrix;
    emu "2" routes every GEMM with K >= 256 (triangular operands included)
    through the INT8 emulation."""
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    monkeypatch.setenv("SKB_GEMM_EMU", emu)
    g = np.random.Generator(np.random.Philox(Mp))
    X = g.standard_normal((Mp + 200, Mp))
    S = X.T @ X
    G = _t(np.tril(S))
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, Mp + 200)))
    _lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr())
    L = np.tril(_h(G))
    assert int(st.item()) == 0
    Lref = np.linalg.cholesky(S)
    assert np.max(np.abs(L - Lref)) <= 1e-10 * np.abs(Lref).max()
    Li = torch.zeros_like(G)
    _lib.call("skb_trtri", G, Li, Mp, Mp, ws, cap, stream_ptr())
    E = np.tril(_h(Li)) @ Lref - np.eye(Mp)
    assert np.max(np.abs(E)) <= 1e-9


@pytest.mark.parametrize("Mp", [64, 192, 1024, 2048, 6144])
def test_potrf_fused_steps_bitwise_equal_panel_loop(K, monkeypatch, Mp):
    """The one-launch-per-panel Cholesky (potrf_step_kernel) against the
    three-launch GEMM panel loop (SKB_POTRF_LOOP=1): same DMMA k sequence and
    epilogue rounding, so L must be bitwise identical; a non-SPD input flags
    the status word in both."""
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    monkeypatch.setenv("SKB_GEMM_EMU", "0")
    g = np.random.Generator(np.random.Philox(Mp + 7))
    X = g.standard_normal((Mp + 64, Mp))
    S = np.tril(X.T @ X)
    ws, cap = workspace(int(_lib.lib().skb_factor_workspace_bytes(Mp, Mp + 64)))
    outs = {}
    for loop in ("0", "1"):
        monkeypatch.setenv("SKB_POTRF_LOOP", loop)
        G = _t(S)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("skb_potrf", G, Mp, Mp, st, ws, cap, stream_ptr())
        assert int(st.item()) == 0
        outs[loop] = _h(G)
    assert np.array_equal(outs["0"], outs["1"])
    assert np.array_equal(np.triu(outs["0"], 1), np.zeros((Mp, Mp)))
    Lref = np.linalg.cholesky(X.T @ X)
    assert np.max(np.abs(outs["0"] - Lref)) <= 1e-10 * np.abs(Lref).max()
    bad = S.copy()
    bad[Mp // 2, Mp // 2] = -1.0
    for loop in ("0", "1"):
        monkeypatch.setenv("SKB_POTRF_LOOP", loop)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("skb_potrf", _t(bad), Mp, Mp, st, ws, cap, stream_ptr())
        assert int(st.item()) & 4


@pytest.mark.parametrize("m,n,mode", [(37, 3001, "feasible"), (100, 5000, "infeasible"),
                                      (512, 20000, "feasible"), (1000, 50001, "infeasible"),
                                      (1500, 20001, "feasible"), (2000, 30000, "infeasible")])
def test_directions_v_fused_bitwise(K, m, n, mode):
    """skb_directions_v (assemble_directions + the v-invariant's A (v / s) in one
    pass, z from shared memory; m > 1024 through the warp-pair kernel) against
    skb_directions and skb_gemv_ratio: every output bitwise identical."""
    g, A = _problem(m, n, m + 11)
    x, s = g.random(n) + 0.2, g.random(n) + 0.2
    dy, v = g.standard_normal(m), 1e-3 * g.standard_normal(n)
    r_d = _t(1e-2 * g.standard_normal(n)) if mode == "infeasible" else None
    Ad = K.DeviceMatrix.from_host(A)
    e = lambda k: torch.empty(k, dtype=torch.float64, device="cuda")  # noqa: E731
    ref = [e(n), e(n), e(m), e(n), e(m)]
    K.directions(Ad, _t(dy), _t(x), _t(s), _t(v), 0.123, ref[0], ref[1], ref[2], atdy=ref[3],
                 r_d=r_d)
    K.gemv_ratio(Ad, _t(v), _t(s), ref[4])
    out = [e(n), e(n), e(m), e(n), e(m)]
    assert K.directions_v(Ad, _t(dy), _t(x), _t(s), _t(v), 0.123, out[0], out[1], out[2],
                          out[4], atdy=out[3], r_d=r_d)
    for a, b in zip(out, ref):
        assert np.array_equal(_h(a), _h(b))


@pytest.mark.parametrize("m,n,mode", [(37, 3001, "feasible"), (1000, 50001, "infeasible"),
                                      (1000, 20000, "feasible"), (2000, 30000, "infeasible")])
def test_iterate_rhs_fused_bitwise(K, m, n, mode):
    """The iterate pass fused with the next step's rhs (skb_step_xs + sigma mu on
    the device + skb_iterate_rhs) against skb_iterate followed by skb_rhs at the
    new point with the host's sigma * mu: x_new, s_new, r_p, r_d and p bitwise."""
    from paper_2209_08722_b200 import _lib
    from paper_2209_08722_b200.lp_model import DeviceLP, LinearProgram
    from paper_2209_08722_b200.runtime import stream_ptr, to_host
    g, A = _problem(m, n, m + 5)
    x, s = g.random(n) + 0.2, g.random(n) + 0.2
    dx, ds = 0.1 * g.standard_normal(n), 0.1 * g.standard_normal(n)
    y = g.standard_normal(m)
    b, c = g.standard_normal(m), g.standard_normal(n)
    lp = DeviceLP.from_host(LinearProgram(A, b, c))
    alpha, sigma = 0.8125, 0.5
    inf = mode == "infeasible"
    fused = lp.iterate_with_rhs(_t(x), _t(s), _t(y), _t(dx), _t(ds), alpha, sigma, inf)
    assert fused is not None
    xo, so, r_p, r_d = lp.iterate(_t(x), _t(s), _t(y), dx=_t(dx), ds=_t(ds), alpha=alpha)
    st = torch.zeros(5, dtype=torch.float64, device="cuda")
    from paper_2209_08722_b200.lp_model import reduce_call
    st = reduce_call("skb_iter_stats", 5, xo, so, None, xo.numel())
    mu = float(to_host(st)[0]) / n
    p = lp.rhs(xo, so, sigma * mu, r_d=r_d if inf else None, r_p=r_p if inf else None)
    for a, bb in zip(fused, (xo, so, r_p, r_d, p)):
        assert np.array_equal(_h(a), _h(bb))
