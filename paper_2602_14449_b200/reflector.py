"""Generalized Householder reflector API (reflector.py of the reference).

The reflector H = I - W T^{-1} W^* is constructed on the GPU from the k0 x k0
top block of V (seed kernels in csrc/small.cu).  In this build the
reflector objects are produced and consumed inside `two_stage_qr`; the
standalone pieces exposed here are `modified_lu` (Algorithm 2) and the
record types."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import errors as E
from ._native import check, lib
from .core import as_matrix, is_complex

CHOICES = ("mlu", "qr", "polar", "explicit")   # reflector.py:41


@dataclass
class MLUResult:
    """reflector.py:44-50."""
    p_diag: object
    l: object
    u_tri: object


@dataclass
class ReflectorDiagnostics:
    """reflector.py:168-171."""
    kappa_t: float
    wt_inv_norm: float


@dataclass
class GenHouseholder:
    """reflector.py:156-165 (record shape kept for drop-in callers)."""
    w: object
    t_solver: object
    p: object
    choice: str
    n: int
    k0: int


def modified_lu(z):
    """Pivot-free LU of diag(p) - z with on-the-fly signs (reflector.py:53-77,
    PAPER Alg. 2), on the GPU.  NormBoundError if ||z||_2 > 1 + 1e-8."""
    was_torch = D.is_torch(z)
    z = as_matrix(z, "z")
    k = z.shape[0]
    if z.shape[0] != z.shape[1]:
        raise E.DimensionError(f"modified_lu needs a square matrix, got {tuple(z.shape)}")
    if is_complex(z):
        raise NotImplementedError("complex modified_lu: not in this build")
    if k == 0:
        e = np.zeros((0, 0))
        return MLUResult(np.ones(0), e, e)
    dev = D.pick_device(z)
    ctx = D.ctx(dev)
    Z = D.to_device(z, dev)
    t = D.torch()
    LU = t.empty((k, k), dtype=t.float64, device=f"cuda:{dev}")
    p = t.empty((k,), dtype=t.float64, device=f"cuda:{dev}")
    import ctypes as C
    rc = lib().ots_modified_lu_f64(ctx, k, Z.ptr, Z.ld, C.c_void_p(LU.data_ptr()),
                                   C.c_void_p(p.data_ptr()), D.stream_ptr(dev))
    check(rc, ctx)
    lo = t.tril(LU, -1) + t.eye(k, dtype=t.float64, device=LU.device)
    up = t.triu(LU)
    if was_torch:
        return MLUResult(p, lo, up)
    return MLUResult(p.cpu().numpy(), lo.cpu().numpy(), up.cpu().numpy())
