"""ctypes binding of libskb.so (the C ABI declared in include/skb.h).

The argument types are read from the header itself, so the binding and the
declared ABI cannot drift apart. There is no CPU fallback: importing the
product path without the built library, or calling it without a CUDA device,
raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
HEADER = os.path.join(ROOT, "include", "skb.h")
LIBPATH = os.path.join(HERE, "libskb.so")

_CTYPES = {
    "int": ctypes.c_int,
    "int32_t": ctypes.c_int32,
    "int64_t": ctypes.c_int64,
    "uint32_t": ctypes.c_uint32,
    "uint64_t": ctypes.c_uint64,
    "size_t": ctypes.c_size_t,
    "double": ctypes.c_double,
    "void": None,
}


class SkbError(DeviceError):
    """A libskb call returned a negative SKB_ERR_* code (a SkipmError, so the
    reference CLI's `except SkipmError` maps it to its numeric exit code)."""

    NAMES = {-1: "SKB_ERR_ARG", -2: "SKB_ERR_DIMS", -3: "SKB_ERR_WORKSPACE",
             -4: "SKB_ERR_CUDA", -5: "SKB_ERR_INTERNAL", -6: "SKB_ERR_UNSUPPORTED"}

    def __init__(self, fn: str, code: int):
        self.code = code
        super().__init__(f"{fn} failed: {self.NAMES.get(code, code)}")


def parse_header(path: str = HEADER) -> dict:
    """-> {name: (restype, [argtypes])} for every prototype in skb.h."""
    with open(path) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
    text = re.sub(r"//[^\n]*", " ", text)
    protos = {}
    for m in re.finditer(r"\b(int32_t|int64_t|int|size_t|void)\s+(skb_\w+)\s*\(([^)]*)\)\s*;", text):
        ret, name, args = m.group(1), m.group(2), m.group(3)
        argtypes = []
        for a in [a.strip() for a in args.split(",") if a.strip() and a.strip() != "void"]:
            if "*" in a:
                argtypes.append(ctypes.c_void_p)
                continue
            toks = a.replace("const", " ").split()
            argtypes.append(_CTYPES[toks[0]])
        protos[name] = (_CTYPES[ret], argtypes)
    return protos


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIBPATH):
            raise ImportError(
                f"{LIBPATH} is missing: build it with `python -m paper_2209_08722_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIBPATH)
        for name, (res, args) in parse_header().items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _arg(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a


def call(name: str, *args) -> int:
    """Call skb_<name>; tensors become device pointers, None becomes NULL."""
    fn = getattr(lib(), name)
    rc = fn(*[_arg(a) for a in args])
    if fn.restype is ctypes.c_int and rc < 0:
        raise SkbError(name, rc)
    return rc
