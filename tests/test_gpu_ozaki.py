"""FP64 GEMM emulated on the INT8 tensor cores (csrc/skb_ozaki.cu) against an
extended-precision reference, and through skb_gemm's routing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_08722_b200 import _lib
    return _lib


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _exact(opa, opb):
    return (opa.astype(np.longdouble) @ opb.astype(np.longdouble))


def _bound(opa, opb):
    """Truncation of each operand row/column at 2^-53 of its max magnitude,
    plus the final rounding: 2^-51 (rowmax_i sum_k |b_kj| + colmax_j sum_k |a_ik|)."""
    ra = np.abs(opa).max(axis=1)[:, None]
    cb = np.abs(opb).max(axis=0)[None, :]
    return 2.0 ** -51 * (ra * np.abs(opb).sum(axis=0)[None, :] + cb * np.abs(opa).sum(axis=1)[:, None])


@pytest.mark.parametrize("M,N,K", [(200, 130, 3000), (64, 300, 1025), (513, 257, 5000)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_ozaki_against_extended(L, M, N, K, ta, tb):
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(M + 3 * N + K + ta + 2 * tb))
    opa = g.standard_normal((M, K)) * np.exp(g.uniform(-3, 3, (M, 1)))
    opb = g.standard_normal((K, N)) * np.exp(g.uniform(-3, 3, (1, N)))
    A = opa.T.copy() if ta else opa.copy()
    B = opb.T.copy() if tb else opb.copy()
    C0 = g.standard_normal((M, N))
    Cd = _t(C0)
    need = int(L.lib().skb_gemm_ozaki_workspace_bytes(M, N, K))
    ws, cap = workspace(need)
    L.call("skb_gemm_ozaki", ta, tb, M, N, K, 0.75, _t(A), A.shape[1], _t(B), B.shape[1], -0.5,
           Cd, N, 0, ws, cap, stream_ptr())
    out = Cd.cpu().numpy()
    ref = 0.75 * _exact(opa, opb) - 0.5 * C0.astype(np.longdouble)
    err = np.abs(out - ref).astype(np.float64)
    bnd = 0.75 * _bound(opa, opb) + 2.0 ** -52 * np.abs(ref).astype(np.float64)
    assert np.all(err <= bnd), float((err / bnd).max())


def test_ozaki_wide_dynamic_range_zero_rows_and_lower(L):
    """Rows spanning 1e-150..1e150, an all-zero row, lower_only writes j <= i."""
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(5))
    M, K = 300, 2000
    X = g.standard_normal((M, K)) * 10.0 ** g.uniform(-150, 150, (M, 1))
    X *= np.exp(g.uniform(-8, 8, (1, K)))  # column dynamic range inside each row
    X[7] = 0.0
    G = torch.full((M, M), 3.0, dtype=torch.float64, device="cuda")
    ws, cap = workspace(int(L.lib().skb_gemm_ozaki_workspace_bytes(M, M, K)))
    L.call("skb_gemm_ozaki", 0, 1, M, M, K, 1.0, _t(X), K, _t(X), K, 0.0, G, M, 1, ws, cap,
           stream_ptr())
    out = G.cpu().numpy()
    ref = _exact(X, X.T)
    low = np.tril(np.ones((M, M), bool))
    err = np.abs(out - ref).astype(np.float64)
    bnd = _bound(X, X.T) + 2.0 ** -52 * np.abs(ref).astype(np.float64)
    assert np.all(err[low] <= bnd[low])
    assert np.all(out[~low] == 3.0)  # untouched above the diagonal
    assert np.all(out[7, :8] == 0.0)


def test_ozaki_deterministic_and_chunked(L, monkeypatch):
    """Integer products: identical bits run to run; a small workspace forces
    K chunks (fp64 accumulation) that stay within the same bound."""
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(9))
    M, N, K = 256, 192, 20000
    A = g.standard_normal((M, K))
    B = g.standard_normal((K, N))
    outs = []
    for cap_div in (1, 1, 6):
        need = int(L.lib().skb_gemm_ozaki_workspace_bytes(M, N, K))
        small = (32 << 20) + 16 * (M + N) * (K // cap_div) + 16 * M * N * 4 + (1 << 20)
        ws, cap = workspace(need if cap_div == 1 else small)
        C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
        L.call("skb_gemm_ozaki", 0, 0, M, N, K, 1.0, _t(A), K, _t(B), N, 0.0, C, N, 0, ws,
               cap if cap_div == 1 else small, stream_ptr())
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    ref = _exact(A, B)
    bnd = 2 * _bound(A, B) + 2.0 ** -51 * np.abs(ref).astype(np.float64)
    for o in (outs[0], outs[2]):
        assert np.all(np.abs(o - ref).astype(np.float64) <= bnd)


def test_skb_gemm_routes_large_products(L, monkeypatch):
    """SKB_GEMM_EMU=2 sends an eligible skb_gemm (incl. kscale via
    skb_weighted_gram) through the emulation; results match DMMA closely."""
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(17))
    m, n = 300, 6000
    A = g.standard_normal((m, n))
    wts = g.random(n) + 0.1
    outs = {}
    for mode in ("0", "2"):
        monkeypatch.setenv("SKB_GEMM_EMU", mode)
        c0 = L.lib().skb_gemm_ozaki_calls()
        G = torch.zeros((m, m), dtype=torch.float64, device="cuda")
        ws, cap = workspace(int(L.lib().skb_gemm_ozaki_workspace_bytes(m, m, n)) + (64 << 20))
        L.call("skb_weighted_gram", _t(A.T), m, n, m, _t(wts), G, m, ws, cap, stream_ptr())
        outs[mode] = np.tril(G.cpu().numpy())
        assert L.lib().skb_gemm_ozaki_calls() - c0 == (1 if mode == "2" else 0)
    ref = (A * wts) @ A.T
    scale = np.abs(ref).max()
    assert np.max(np.abs(outs["2"] - np.tril(ref))) <= 1e-13 * scale
    assert np.max(np.abs(outs["2"] - outs["0"])) <= 1e-13 * scale


def test_ozaki_nonfinite_rows_and_empty_k(L):
    """A NaN / inf in an operand row poisons only that output row (NaN), as in
    fp64; K = 0 gives beta C."""
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(21))
    M, N, K = 64, 48, 700
    A = g.standard_normal((M, K))
    B = g.standard_normal((K, N))
    A[3, 10] = np.nan
    A[7, 0] = np.inf
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    ws, cap = workspace(int(L.lib().skb_gemm_ozaki_workspace_bytes(M, N, K)))
    L.call("skb_gemm_ozaki", 0, 0, M, N, K, 1.0, _t(A), K, _t(B), N, 0.0, C, N, 0, ws, cap,
           stream_ptr())
    out = C.cpu().numpy()
    assert np.isnan(out[3]).all() and np.isnan(out[7]).all()
    ok = np.ones(M, bool)
    ok[[3, 7]] = False
    ref = _exact(A[ok], B)
    assert np.all(np.abs(out[ok] - ref).astype(np.float64) <= _bound(A[ok], B) + 1e-300)
    C0 = g.standard_normal((M, N))
    Cd = _t(C0)
    L.call("skb_gemm_ozaki", 0, 0, M, N, 0, 1.0, _t(A), K, _t(B), N, 0.5, Cd, N, 0, ws, cap,
           stream_ptr())
    assert np.array_equal(Cd.cpu().numpy(), 0.5 * C0)


def test_ozaki_thread_pool_matches_sequential(L):
    """Concurrent host threads (run_comparison's ThreadPoolExecutor pattern)
    share the cuBLASLt handle: results stay bitwise equal to sequential calls."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    shapes = [(300, 200, 3000), (128, 512, 2048), (700, 333, 1500), (64, 64, 5000)]
    data = []
    for i, (M, N, K) in enumerate(shapes):
        g = np.random.Generator(np.random.Philox(100 + i))
        data.append((g.standard_normal((M, K)), g.standard_normal((K, N))))

    def run(i):
        M, N, K = shapes[i]
        A, B = data[i]
        C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
        ws, cap = workspace(int(L.lib().skb_gemm_ozaki_workspace_bytes(M, N, K)))
        L.call("skb_gemm_ozaki", 0, 0, M, N, K, 1.0, _t(A), K, _t(B), N, 0.0, C, N, 0, ws, cap,
               stream_ptr())
        torch.cuda.current_stream().synchronize()
        return C.cpu().numpy()

    alone = [run(i) for i in range(len(shapes))]
    with ThreadPoolExecutor(max_workers=4) as pool:
        together = list(pool.map(run, range(len(shapes))))
    for a, b in zip(alone, together):
        assert np.array_equal(a, b)
