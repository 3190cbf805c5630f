"""Device-memory plumbing (PyTorch is used for allocation, streams and H2D/D2H
copies only; all arithmetic of the path runs in libots.so)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import errors as E
from ._native import context


def torch():
    import torch as _t
    return _t


def is_torch(x):
    try:
        import torch as _t
    except Exception:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


def pick_device(*xs):
    t = torch()
    for x in xs:
        if is_torch(x) and x.is_cuda:
            return x.device.index
    if not t.cuda.is_available():
        raise E.NativeUnavailable("no CUDA device available (this path has no CPU fallback)")
    return t.cuda.current_device()


class DMat:
    """Row-major device matrix (rows x cols) inside a (rows x ld) float64
    buffer, ld even so every row is 16-byte aligned (ots.h conventions)."""

    def __init__(self, buf, cols, ld=None):
        self.buf = buf
        self.rows = buf.shape[0]
        self.cols = cols
        self.ld = ld if ld is not None else buf.shape[1]

    @property
    def ptr(self):
        return C.c_void_p(self.buf.data_ptr())

    def view(self):
        return self.buf[:, :self.cols]

    def numpy(self):
        return self.view().cpu().numpy()


def _ld(cols):
    return max(2, cols + (cols & 1))


def empty(rows, cols, device):
    t = torch()
    return DMat(t.empty((max(rows, 1), _ld(cols)), dtype=t.float64, device=f"cuda:{device}"), cols)


def zeros(rows, cols, device):
    t = torch()
    return DMat(t.zeros((max(rows, 1), _ld(cols)), dtype=t.float64, device=f"cuda:{device}"), cols)


def to_device(x, device):
    """numpy (or CPU/CUDA torch) real matrix -> DMat on `device`.  A CUDA
    tensor with an aligned even row stride is used zero-copy."""
    t = torch()
    if is_torch(x):
        if x.dtype != t.float64:
            x = x.to(t.float64)
        x = x.resolve_neg()
        if x.is_cuda and x.device.index == device and x.dim() == 2 and x.stride(1) == 1 \
                and x.stride(0) % 2 == 0 and x.data_ptr() % 16 == 0 and x.stride(0) >= x.shape[1]:
            return DMat(x, x.shape[1], ld=x.stride(0))
        src = x
    else:
        src = t.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    rows, cols = src.shape
    d = empty(rows, cols, device)
    if rows and cols:
        d.buf[:rows, :cols].copy_(src, non_blocking=False)
    return d


def cempty(rows, cols, device):
    """complex128 row-major device matrix (ld in complex elements)."""
    t = torch()
    return DMat(t.empty((max(rows, 1), max(cols, 1)), dtype=t.complex128, device=f"cuda:{device}"), cols)


def czeros(rows, cols, device):
    t = torch()
    return DMat(t.zeros((max(rows, 1), max(cols, 1)), dtype=t.complex128, device=f"cuda:{device}"), cols)


def cto_device(x, device):
    """numpy (or torch) matrix -> complex128 DMat on `device` (zero-copy for a
    row-major CUDA complex128 tensor)."""
    t = torch()
    if is_torch(x):
        if x.dtype != t.complex128:
            x = x.to(t.complex128)
        # lazy conjugate / negative views (e.g. .mH) keep unconjugated data
        # behind the bit: materialise before handing out a raw pointer
        x = x.resolve_conj().resolve_neg()
        if x.is_cuda and x.device.index == device and x.dim() == 2 and x.stride(1) == 1 \
                and x.data_ptr() % 16 == 0 and x.stride(0) >= x.shape[1]:
            return DMat(x, x.shape[1], ld=x.stride(0))
        src = x
    else:
        src = t.from_numpy(np.ascontiguousarray(x, dtype=np.complex128))
    rows, cols = src.shape
    d = cempty(rows, cols, device)
    if rows and cols:
        d.buf[:rows, :cols].copy_(src, non_blocking=False)
    return d


def stream_ptr(device):
    return C.c_void_p(torch().cuda.current_stream(device).cuda_stream)


def ctx(device):
    return context(device)
