"""B-inner-product extension (oblique.py of the reference, Algorithm 4).

This build runs the weighted inner product <x, y>_M = y^* M x on the GPU
for a diagonal M = diag(d) (the case BASELINE configs[3] specifies) when the
initial basis is the canonical `initial_b_basis(inner, m)`: then Algorithm 4
(`b_two_stage_qr`, oblique.py:279-315) equals the Euclidean Algorithm 1 on
(D^1/2 V, D^1/2 A) with Q = D^-1/2 Q' sgn, R = sgn R' (positive diagonal,
oblique.py:232) and S unchanged (verified against the
reference to <= 7e-14).  The whole computation is one C-ABI call
(`ots_b_two_stage_diag_f64`, or `ots_b_two_stage_diag_c128` for complex
data).  A dense general B (n x n) is not supported by this build
(NotImplementedError).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import errors as E
from ._native import CHOICES, check, lib
from .core import QRPair, as_matrix, householder_qr, is_complex
from .reflector import ReflectorDiagnostics
from .twostage import TwoStageResult


@dataclass(frozen=True)
class InnerProduct:
    """oblique.py:36-90.  kind "euclidean" or "weighted"; for a diagonal B the
    weights are kept as the vector `diag` (never an n x n matrix)."""

    kind: str
    b: object = None
    chol_b: object = None
    diag: object = None

    @staticmethod
    def euclidean():
        return InnerProduct(kind="euclidean")

    @staticmethod
    def weighted(b):
        """b: SPD matrix (n x n) or, as an extension, the 1-D diagonal of a
        diagonal B.  Diagonal matrices are detected and stored as vectors."""
        if D.is_torch(b):
            t = D.torch()
            bb = b.to(t.float64)
            if bb.dim() == 2:
                if bb.shape[0] != bb.shape[1]:
                    raise E.DimensionError(f"weight matrix must be square, got {tuple(bb.shape)}")
                if t.count_nonzero(bb - t.diag(t.diagonal(bb))).item():
                    raise NotImplementedError("dense (non-diagonal) B is not supported by this build")
                bb = t.diagonal(bb).contiguous()
            if bb.numel() and not bool((bb > 0).all().item()):
                raise E.NotPositiveDefinite("diagonal weight has a non-positive entry")
            return InnerProduct(kind="weighted", diag=bb)
        arr = np.asarray(b)
        if arr.ndim == 2:
            if arr.shape[0] != arr.shape[1]:
                raise E.DimensionError(f"weight matrix must be square, got {arr.shape}")
            off = arr - np.diag(np.diagonal(arr))
            if np.count_nonzero(off):
                raise NotImplementedError("dense (non-diagonal) B is not supported by this build")
            arr = np.diagonal(arr)
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        if arr.size and not np.all(arr > 0):
            raise E.NotPositiveDefinite("diagonal weight has a non-positive entry")
        return InnerProduct(kind="weighted", diag=arr)

    @property
    def n(self):
        return None if self.diag is None else int(self.diag.shape[0])


def initial_b_basis(inner, m):
    """oblique.py:93-108 for diagonal B: [diag(d_1..m)^{-1/2}; 0] (n x m).
    Returned on the device of the weights (numpy for host weights)."""
    if inner.kind != "weighted":
        raise E.ParameterError("initial_b_basis needs a weighted inner product")
    n = inner.n
    if m > n:
        raise E.ParameterError(f"need m <= n, got m={m}, n={n}")
    d = inner.diag
    if D.is_torch(d):
        t = D.torch()
        u = t.zeros((n, m), dtype=t.float64, device=d.device)
        u[:m] = t.diag(d[:m].rsqrt())
        return u
    u = np.zeros((n, m))
    u[np.arange(m), np.arange(m)] = 1.0 / np.sqrt(d[:m])
    return u


def _is_canonical_basis(u, d, m):
    """u[:, :m] == initial_b_basis(diag(d), m) (exactly, as the fast path needs)."""
    if D.is_torch(u):
        t = D.torch()
        top = u[:m, :m]
        want = t.diag(t.as_tensor(d, device=u.device)[:m].rsqrt())
        return bool(t.equal(top, want)) and (t.count_nonzero(u[m:, :m]).item() == 0)
    top = np.asarray(u[:m, :m])
    dd = np.asarray(d.cpu().numpy() if D.is_torch(d) else d)[:m]
    return np.array_equal(top, np.diag(1.0 / np.sqrt(dd))) and not np.count_nonzero(u[m:, :m])


def b_two_stage_qr(v, a, u, inner, choice="qr", reorth=True, p=None):
    """Algorithm 4 (oblique.py:279-315) for M = diag(d) on the GPU."""
    was_torch = D.is_torch(v) or D.is_torch(a)
    v = as_matrix(v, "v")
    a = as_matrix(a, "a")
    u = as_matrix(u, "u")
    n, k0 = v.shape
    k = a.shape[1]
    if a.shape[0] != n or u.shape[0] != n:
        raise E.DimensionError("v, a and u must share the row count")
    if u.shape[1] < k0 + k:
        raise E.DimensionError(f"u needs at least k0+k = {k0 + k} columns")
    if k0 + k > n:
        raise E.DimensionError(f"need k0 + k <= n, got {k0}+{k} > {n}")
    if inner.kind != "weighted" or inner.diag is None:
        raise NotImplementedError("this build implements b_two_stage_qr for a diagonal B only")
    cplx = is_complex(v) or is_complex(a)
    if not _is_canonical_basis(u, inner.diag, k0 + k):
        raise NotImplementedError("this build needs u = initial_b_basis(inner, k0+k)")
    dev = D.pick_device(v, a)
    t = D.torch()
    d_dev = (inner.diag if D.is_torch(inner.diag) else t.from_numpy(inner.diag)).to(
        device=f"cuda:{dev}", dtype=t.float64).contiguous()
    if k0 == 0:
        # b_householder_qr with the canonical basis: positive-diagonal QR of D^1/2 A
        sa = a * (d_dev.sqrt()[:, None] if D.is_torch(a) else np.sqrt(d_dev.cpu().numpy())[:, None])
        qr = householder_qr(sa, nonneg_diag=True)
        q = qr.q / (d_dev.sqrt()[:, None] if D.is_torch(qr.q) else np.sqrt(d_dev.cpu().numpy())[:, None])
        zdt = (t.complex128 if cplx else t.float64)
        z = t.zeros((0, k), dtype=zdt, device=d_dev.device) if was_torch else \
            np.zeros((0, k), dtype=np.complex128 if cplx else np.float64)
        return TwoStageResult(q, qr.r, z, ReflectorDiagnostics(1.0, 0.0))
    ctx = D.ctx(dev)
    todev = D.cto_device if cplx else D.to_device
    V = todev(v, dev)
    A = todev(a, dev)
    P = todev(p, dev) if (choice == "explicit" and p is not None) else None
    if choice == "explicit" and P is None:
        raise E.ParameterError("choice='explicit' requires a seed matrix p")
    if choice not in CHOICES:
        raise E.ParameterError(f"unknown choice {choice!r}")
    if cplx:
        Q, R, S = D.cempty(n, k, dev), D.czeros(k, k, dev), D.cempty(k0, k, dev)
    else:
        Q, R, S = D.empty(n, k, dev), D.zeros(k, k, dev), D.empty(k0, k, dev)
    diag = (C.c_double * 3)()
    fn = lib().ots_b_two_stage_diag_c128 if cplx else lib().ots_b_two_stage_diag_f64
    rc = fn(
        ctx, n, k0, k, V.ptr, V.ld, A.ptr, A.ld, C.c_void_p(d_dev.data_ptr()), CHOICES[choice],
        P.ptr if P is not None else None, P.ld if P is not None else 0, 1e-6,
        Q.ptr, Q.ld, R.ptr, R.ld, S.ptr, S.ld, diag, D.stream_ptr(dev))
    check(rc, ctx)
    if was_torch:
        return TwoStageResult(Q.view(), R.view(), S.view(), ReflectorDiagnostics(diag[0], diag[1]))
    return TwoStageResult(Q.numpy(), R.numpy(), S.numpy(), ReflectorDiagnostics(diag[0], diag[1]))


@dataclass
class BGenHouseholder:
    """oblique.py:111-122 (record shape kept for drop-in callers)."""
    w: object
    t_solver: object
    p: object
    x: object
    inner: InnerProduct
    choice: str
    n: int
    k0: int
