"""Dense-core entry points of the drop-in API (core.py of the reference).

`householder_qr` (core.py:61-84) runs on the GPU: TSQR Householder with
LAPACK dgeqrf/dorgqr sign convention recovered exactly (chainqr.cu +
small.cu sign kernel).  `as_matrix` mirrors core.py:25-32 for host arrays and
accepts CUDA tensors unchanged (zero-copy path)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import errors as E
from ._native import check, lib

EPS = 2.0 ** -53  # core.py:22


def as_matrix(a, name="matrix"):
    """core.py:25-32: 2-D check; float64/complex128.  CUDA tensors pass
    through (dtype-cast only)."""
    if D.is_torch(a):
        if a.dim() != 2:
            raise E.DimensionError(f"{name} must be 2-D, got shape {tuple(a.shape)}")
        t = D.torch()
        if a.is_complex():
            return a.to(t.complex128)
        return a.to(t.float64)
    a = np.asarray(a)
    if a.ndim != 2:
        raise E.DimensionError(f"{name} must be 2-D, got shape {a.shape}")
    if np.iscomplexobj(a):
        return np.ascontiguousarray(a, dtype=np.complex128)
    return np.ascontiguousarray(a, dtype=np.float64)


def is_complex(x):
    return x.is_complex() if D.is_torch(x) else np.iscomplexobj(x)


def all_finite(x):
    if D.is_torch(x):
        return bool(D.torch().isfinite(x).all().item()) if x.numel() else True
    return bool(np.all(np.isfinite(x))) if x.size else True


def out_like(inputs_torch, dmat):
    """numpy in -> numpy out; torch in -> torch (device) out."""
    return dmat.view() if inputs_torch else dmat.numpy()


@dataclass
class QRPair:
    """core.py:52-58."""
    q: object
    r: object


def householder_qr(a, nonneg_diag=False):
    """QR of a tall matrix on the GPU (core.py:61-84 semantics)."""
    was_torch = D.is_torch(a)
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise E.DimensionError(f"need rows >= cols, got {m}x{n}")
    if not all_finite(a):
        raise ValueError("input contains non-finite entries")
    dev = D.pick_device(a)
    ctx = D.ctx(dev)
    if is_complex(a):
        A = D.cto_device(a, dev)
        Q = D.cempty(m, n, dev)
        R = D.czeros(n, n, dev)
        if n:
            rc = lib().ots_householder_qr_c128(ctx, m, n, A.ptr, A.ld, Q.ptr, Q.ld, R.ptr, R.ld,
                                               1 if nonneg_diag else 0, D.stream_ptr(dev))
            check(rc, ctx)
        return QRPair(out_like(was_torch, Q), out_like(was_torch, R))
    A = D.to_device(a, dev)
    Q = D.empty(m, n, dev)
    R = D.zeros(n, n, dev)
    if n:
        rc = lib().ots_householder_qr_f64(ctx, m, n, A.ptr, A.ld, Q.ptr, Q.ld, R.ptr, R.ld,
                                          1 if nonneg_diag else 0, D.stream_ptr(dev))
        check(rc, ctx)
    return QRPair(out_like(was_torch, Q), out_like(was_torch, R))


def shifted_cholesky_qr(a, refine_passes=2):
    """Shifted Cholesky-QR + 2 unshifted refinements on the GPU
    (core.py:177-202).  Breakdown raises NotPositiveDefinite."""
    if refine_passes != 2:
        raise NotImplementedError("this build implements the reference's 2 refinement passes")
    was_torch = D.is_torch(a)
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise E.DimensionError(f"need rows >= cols, got {m}x{n}")
    dev = D.pick_device(a)
    ctx = D.ctx(dev)
    if is_complex(a):
        A = D.cto_device(a, dev)
        Q = D.cempty(m, n, dev)
        R = D.czeros(n, n, dev)
        if n:
            rc = lib().ots_shifted_cholesky_qr_c128(ctx, m, n, A.ptr, A.ld, Q.ptr, Q.ld, R.ptr, R.ld,
                                                    D.stream_ptr(dev))
            check(rc, ctx)
        return QRPair(out_like(was_torch, Q), out_like(was_torch, R))
    A = D.to_device(a, dev)
    Q = D.empty(m, n, dev)
    R = D.zeros(n, n, dev)
    if n:
        rc = lib().ots_shifted_cholesky_qr_f64(ctx, m, n, A.ptr, A.ld, Q.ptr, Q.ld, R.ptr, R.ld,
                                               D.stream_ptr(dev))
        check(rc, ctx)
    return QRPair(out_like(was_torch, Q), out_like(was_torch, R))
