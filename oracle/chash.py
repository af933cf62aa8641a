"""ORACLE — test infrastructure only (see oracle/__init__.py).

ctypes view of oracle/philox_hash.c (built by oracle/Makefile or
__graft_entry__.build())."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_hash.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle_hash.so"], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "philox_hash.c")
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(_SO)
        u64, i64, i32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32
        P = ctypes.c_void_p
        L.oracle_out64.restype = u64
        L.oracle_out64.argtypes = [u64, u64, u64]
        L.oracle_lemire_draw.restype = None
        L.oracle_lemire_draw.argtypes = [u64, u64, P, ctypes.c_uint32, i64, P]
        L.oracle_sparse_embedding.restype = u64
        L.oracle_sparse_embedding.argtypes = [u64, u64, i64, i32, i32, P, P]
        L.oracle_adw_dense.restype = None
        L.oracle_adw_dense.argtypes = [P, i64, i64, P, P, P, i32, i32, P]
        _lib = L
    return _lib


def philox_key(seed: int):
    k = np.random.SeedSequence(int(seed)).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


def out64(seed: int, k: int) -> int:
    k0, k1 = philox_key(seed)
    return int(lib().oracle_out64(k0, k1, k))


def lemire_draw(seed: int, w: int, cnt: int, pos: int = 0):
    k0, k1 = philox_key(seed)
    out = np.empty(cnt, dtype=np.int64)
    p = ctypes.c_uint64(pos)
    lib().oracle_lemire_draw(k0, k1, ctypes.byref(p), w, cnt, out.ctypes.data)
    return out, int(p.value)


def sparse_embedding(n: int, w: int, s: int, seed: int):
    """-> (cols int64 (n,s), vals f64 (n,s), words consumed); 2s < w only."""
    assert 2 * s < w
    k0, k1 = philox_key(seed)
    cols = np.empty((n, s), dtype=np.int64)
    vals = np.empty((n, s), dtype=np.float64)
    used = lib().oracle_sparse_embedding(k0, k1, n, w, s, cols.ctypes.data, vals.ctypes.data)
    return cols, vals, int(used)


def adw_dense(A: np.ndarray, d: np.ndarray, cols: np.ndarray, vals: np.ndarray, w: int):
    A = np.ascontiguousarray(A, dtype=np.float64)
    m, n = A.shape
    s = cols.shape[1]
    out = np.empty((m, w), dtype=np.float64)
    lib().oracle_adw_dense(A.ctypes.data, m, n, np.ascontiguousarray(d).ctypes.data,
                           np.ascontiguousarray(cols, dtype=np.int64).ctypes.data,
                           np.ascontiguousarray(vals).ctypes.data, s, w, out.ctypes.data)
    return out
