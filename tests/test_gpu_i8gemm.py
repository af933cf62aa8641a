"""The hand-written tcgen05 INT8 GEMM (csrc/skb_i8gemm.cu): exact int32 batch
products against numpy int64, on ragged tiles, row/K offsets and long K; and
the whole FP64 emulation (skb_gemm_ozaki) bit-identical to the same emulation
with cuBLASLt's INT8 kernel in its place (integer products are exact, so any
difference would be a bug in one of the two)."""

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


def _run(L, A, B, Kp, rows, cols, ar0, br0, k0, k1, ldc=None, tri=0, tri_off=0):
    from paper_2209_08722_b200.runtime import stream_ptr
    n, Ra, _ = A.shape
    Rb = B.shape[1]
    ldc = ldc or (cols + 15) // 16 * 16
    Ad = torch.from_numpy(A).cuda()
    Bd = torch.from_numpy(B).cuda()
    C = torch.full((n, rows, ldc), -7, dtype=torch.int32, device="cuda")
    L.call("skb_i8gemm_batched", Ad, Ra, Ra * Kp, Bd, Rb, Rb * Kp, Kp, C, ldc, rows * ldc, rows,
           cols, ar0, br0, k0, k1, n, tri, tri_off, stream_ptr())
    torch.cuda.synchronize()
    return C.cpu().numpy()


CASES = [  # n, Ra, Rb, Kp, rows, cols, ar0, br0, k0, k1
    (1, 128, 256, 128, 128, 256, 0, 0, 0, 128),
    (3, 300, 520, 1024, 300, 512, 0, 0, 0, 1024),
    (16, 700, 600, 640, 257, 336, 33, 17, 128, 544),
    (2, 1000, 900, 4096, 1000, 896, 0, 0, 0, 4096),
    (4, 130, 130, 40960, 130, 128, 0, 2, 0, 40960),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[:6]) for c in CASES])
def test_i8gemm_exact(L, case):
    n, Ra, Rb, Kp, rows, cols, ar0, br0, k0, k1 = case
    g = np.random.Generator(np.random.Philox(sum(case)))
    A = g.integers(-128, 128, (n, Ra, Kp), dtype=np.int8)
    B = g.integers(-128, 128, (n, Rb, Kp), dtype=np.int8)
    # the contract: entries of the 128-rounded K range the caller does not want are zero
    kz = (k1 + 127) // 128 * 128
    A[:, :, k1:kz] = 0
    C = _run(L, A, B, Kp, rows, cols, ar0, br0, k0, k1)
    for l in range(n):
        a = A[l, ar0:ar0 + rows, k0:k1].astype(np.int64)
        b = B[l, br0:br0 + cols, k0:k1].astype(np.int64)
        ref = np.zeros((rows, cols), dtype=np.int64)
        ra, rb = a.shape[0], b.shape[0]
        ref[:ra, :rb] = a @ b.T
        assert np.array_equal(C[l, :, :cols].astype(np.int64), ref), l
        if C.shape[2] > cols:  # padding columns untouched
            assert np.all(C[l, :, cols:] == -7)


@pytest.mark.parametrize("tri_off", [0, 300, -200])
def test_i8gemm_lower_tiles(L, tri_off):
    """tri = 1: every 256-block meeting col <= row + tri_off is exact; blocks
    wholly above that diagonal are untouched, or exact where a wider (512-column)
    pair tile that meets the diagonal covers them."""
    n, R, Kp = 3, 1104, 512
    g = np.random.Generator(np.random.Philox(9 + abs(tri_off)))
    A = g.integers(-128, 128, (n, R, Kp), dtype=np.int8)
    C = _run(L, A, A, Kp, R, R, 0, 0, 0, Kp, tri=1, tri_off=tri_off)
    for l in range(n):
        a = A[l].astype(np.int64)
        ref = a @ a.T
        for i0 in range(0, R, 256):
            for j0 in range(0, R, 256):
                blk = C[l, i0:i0 + 256, j0:j0 + 256]
                if j0 <= i0 + 255 + tri_off:
                    assert np.array_equal(blk, ref[i0:i0 + 256, j0:j0 + 256]), (l, i0, j0)
                else:
                    ok = np.all(blk == -7) or np.array_equal(blk, ref[i0:i0 + 256, j0:j0 + 256])
                    assert ok and (j0 <= i0 + 511 + tri_off or np.all(blk == -7)), (l, i0, j0)


def test_emulated_fp64_gemm_identical_to_cublaslt_route(L, monkeypatch):
    """The emulated FP64 products (full, lower-only, triangular operands via
    skb_gemm's emulation path) are bitwise equal whether the INT8 products run
    on this kernel or on cuBLASLt (SKB_OZ_CUBLASLT=1, development A/B), both with
    the int32-product CRT (SKB_OZ_CRT32=1). The default residue epilogue
    (int8 residues, the CRT reading one byte per product) may represent a
    p = 256 tie as -128 instead of +128 -- the same residue class, another
    split of the same exact integer -- so it agrees to the last bits only."""
    from paper_2209_08722_b200.runtime import stream_ptr, workspace
    g = np.random.Generator(np.random.Philox(77))
    for (M, N, K, lower) in [(700, 500, 3000, 0), (1300, 1300, 2500, 1), (257, 1029, 40000, 0)]:
        A = g.standard_normal((M, K)) * np.exp(g.uniform(-5, 5, (M, 1)))
        B = g.standard_normal((N, K)) * np.exp(g.uniform(-5, 5, (N, 1)))
        C0 = g.standard_normal((M, N))
        outs = []
        for route, crt32 in (("0", "1"), ("1", "1"), ("0", "0")):
            monkeypatch.setenv("SKB_OZ_CUBLASLT", route)
            monkeypatch.setenv("SKB_OZ_CRT32", crt32)
            Cd = torch.from_numpy(C0.copy()).cuda()
            need = int(L.lib().skb_gemm_ozaki_workspace_bytes(M, N, K))
            ws, cap = workspace(need)
            L.call("skb_gemm_ozaki", 0, 1, M, N, K, 1.0, torch.from_numpy(A).cuda(), K,
                   torch.from_numpy(B).cuda(), K, 0.5, Cd, N, lower, ws, cap, stream_ptr())
            torch.cuda.synchronize()
            outs.append(Cd.cpu().numpy())
        assert np.array_equal(outs[0], outs[1]), (M, N, K, lower)
        ref = 0.5 * C0 + A @ B.T
        scale = (np.abs(A) @ np.abs(B).T) + 0.5 * np.abs(C0)
        dres = np.abs(outs[2] - outs[0])
        print(f"[{M}x{N}x{K} lower={lower}] residue-epilogue vs int32 CRT: "
              f"{int(np.count_nonzero(dres))} entries differ, max {float((dres / scale).max()):.1e} "
              f"x (|A||B|' + |beta C|)")
        assert np.all(dres <= 2.0 ** -51 * scale)
        for o in (outs[0], outs[2]):
            if lower:
                il = np.tril_indices(M, 0, N)
                assert np.allclose(o[il], ref[il], rtol=1e-12, atol=1e-10 * np.abs(ref).max())
            else:
                assert np.allclose(o, ref, rtol=1e-12, atol=1e-10 * np.abs(ref).max())


MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


@pytest.mark.parametrize("case", CASES[1:4], ids=[str(c[:6]) for c in CASES[1:4]])
def test_i8gemm_residue_epilogue(L, case):
    """skb_i8gemm_residues: every product stored as its symmetric residue mod p_l
    in int8 (ties of p = 256 as -128), exactly the reduction the CRT applies to
    the int32 products; padding untouched."""
    from paper_2209_08722_b200.runtime import stream_ptr
    n, Ra, Rb, Kp, rows, cols, ar0, br0, k0, k1 = case
    g = np.random.Generator(np.random.Philox(7 + sum(case)))
    A = g.integers(-128, 128, (n, Ra, Kp), dtype=np.int8)
    B = g.integers(-128, 128, (n, Rb, Kp), dtype=np.int8)
    kz = (k1 + 127) // 128 * 128
    A[:, :, k1:kz] = 0
    ldc = (cols + 15) // 16 * 16 + 16
    C8 = torch.full((n, rows, ldc), 99, dtype=torch.int8, device="cuda")
    mod = np.array(MODULI[:n], dtype=np.float64)
    L.call("skb_i8gemm_residues", torch.from_numpy(A).cuda(), Ra, Ra * Kp,
           torch.from_numpy(B).cuda(), Rb, Rb * Kp, Kp, C8, ldc, rows * ldc, rows, cols, ar0, br0,
           k0, k1, n, 0, 0, mod.ctypes.data, stream_ptr())
    torch.cuda.synchronize()
    out = C8.cpu().numpy()
    for l in range(n):
        a = A[l, ar0:ar0 + rows, k0:k1].astype(np.int64)
        b = B[l, br0:br0 + cols, k0:k1].astype(np.int64)
        ref = np.zeros((rows, cols), dtype=np.int64)
        ref[:a.shape[0], :b.shape[0]] = a @ b.T
        p = int(mod[l])
        r = ref - np.round(ref / p).astype(np.int64) * p      # [-p/2, p/2]
        r = np.where(r == 128, -128, r)                        # p = 256 ties
        assert np.array_equal(out[l, :, :cols].astype(np.int64), r), l
        assert np.all(out[l, :, cols:] == 99)
