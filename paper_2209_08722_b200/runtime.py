"""Device plumbing: CUDA device/stream, workspace, pinned scalar readback.

PyTorch is used only as the allocator and stream provider; every arithmetic
operation on the hot path is a libskb kernel.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib

F64 = torch.float64


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_08722_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


class Workspace:
    """Grow-only device scratch buffer shared by consecutive (stream-ordered) calls."""

    def __init__(self):
        self._buf = None
        self._lock = threading.Lock()

    def get(self, nbytes: int):
        with self._lock:
            if self._buf is None or self._buf.numel() < nbytes:
                n = max(int(nbytes), 1 << 20)
                if n <= 1 << 30:
                    n = 1 << (n - 1).bit_length()   # small: powers of two
                else:
                    n = -(-n // (256 << 20)) * (256 << 20)  # large: 256 MB granules
                big = self._buf is not None and self._buf.numel() >= 1 << 30
                self._buf = None  # drop the old buffer before the new one is allocated
                if big:
                    torch.cuda.empty_cache()
                self._buf = torch.empty(n, dtype=torch.uint8, device=require_cuda())
            return self._buf, self._buf.numel()


_WS = threading.local()


def workspace(nbytes: int):
    """-> (tensor, capacity) for the calling thread's workspace."""
    w = getattr(_WS, "ws", None)
    if w is None:
        w = _WS.ws = Workspace()
    return w.get(nbytes)


class Scalars:
    """A small device buffer of doubles read back through pinned memory."""

    def __init__(self, n: int):
        dev = require_cuda()
        self.dev = torch.zeros(n, dtype=F64, device=dev)
        self.host = torch.zeros(n, dtype=F64, pin_memory=True)

    def fetch(self) -> np.ndarray:
        self.host.copy_(self.dev, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.host.numpy().copy()


_PIN = threading.local()


def to_host(t: torch.Tensor) -> np.ndarray:
    """A small device tensor as a host numpy array, through the calling
    thread's pinned staging buffer (a pageable readback costs several times
    the latency, and the solver reads a few scalars back every step)."""
    if not t.is_cuda:
        return t.detach().numpy()
    nbytes = t.numel() * t.element_size()
    buf = getattr(_PIN, "buf", None)
    if buf is None or buf.numel() < nbytes:
        buf = _PIN.buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, pin_memory=True)
    view = buf[:nbytes].view(t.dtype).view(t.shape)
    view.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return view.numpy().copy()


def lda_for(m: int) -> int:
    """Column stride of the device layout: even, so every column is 16-byte aligned."""
    return m + (m & 1)
