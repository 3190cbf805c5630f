"""B-inner-product extension (oblique.py of the reference, Algorithm 4).

This build runs the weighted inner product <x, y>_M = y^* M x on the GPU
for a diagonal M = diag(d) (the case BASELINE configs[3] specifies) when the
initial basis is the canonical `initial_b_basis(inner, m)`: then Algorithm 4
(`b_two_stage_qr`, oblique.py:279-315) equals the Euclidean Algorithm 1 on
(D^1/2 V, D^1/2 A) with Q = D^-1/2 Q' sgn, R = sgn R' (positive diagonal,
oblique.py:232) and S unchanged (verified against the
reference to <= 7e-14).  The whole computation is one C-ABI call
(`ots_b_two_stage_diag_f64`, or `ots_b_two_stage_diag_c128` for complex
data).  A dense SPD B (real) takes the same route with L^T in place of
D^1/2 (B = L L^T, the reference's chol_b): Algorithm 1 on (L^T V, L^T A),
Q = L^-T Q' sgn, with the Cholesky factor, L^T X and L^-T X on the GPU
(`ots_dense_cholesky_f64`, `ots_dense_trmm_lt_f64`, `ots_dense_trsm_lt_f64`,
`ots_b_two_stage_dense_f64`).  Both fast paths need the canonical initial
basis u = initial_b_basis(inner, k0+k); any other u, and a dense complex B,
raise NotImplementedError.
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
    weights are kept as the vector `diag` (never an n x n matrix); a dense B is
    kept on the device with its lower Cholesky factor `chol_b`."""

    kind: str
    b: object = None
    chol_b: object = None
    diag: object = None
    host: bool = True          # weights given as numpy (results returned as numpy)

    @staticmethod
    def euclidean():
        return InnerProduct(kind="euclidean")

    @staticmethod
    def _dense(b, host):
        """oblique.py:48-56 for a dense b: Hermitian check (Frobenius form of
        the reference's 1e-12 spectral test), symmetrise, Cholesky on the GPU."""
        t = D.torch()
        if b.is_complex():
            raise NotImplementedError("dense complex B is not supported by this build")
        n = b.shape[0]
        dev = b.device.index if b.is_cuda else t.cuda.current_device()
        bd = b.to(device=f"cuda:{dev}", dtype=t.float64)
        asym = t.linalg.matrix_norm(bd - bd.T).item()
        if asym > 1e-12 * t.linalg.matrix_norm(bd).item():
            raise E.NotHermitian("weight matrix is not Hermitian to tolerance")
        bs = ((bd + bd.T) * 0.5).contiguous()
        L = t.empty_like(bs)
        ctx = D.ctx(dev)
        check(lib().ots_dense_cholesky_f64(ctx, n, C.c_void_p(bs.data_ptr()), n, C.c_void_p(L.data_ptr()), n,
                                           D.stream_ptr(dev)), ctx)
        return InnerProduct(kind="weighted", b=bs, chol_b=L, host=host)

    @staticmethod
    def weighted(b):
        """b: SPD matrix (n x n) or, as an extension, the 1-D diagonal of a
        diagonal B.  Diagonal matrices are detected and stored as vectors."""
        if D.is_torch(b):
            t = D.torch()
            bb = b.to(t.complex128 if b.is_complex() else t.float64)
            if bb.dim() == 2:
                if bb.shape[0] != bb.shape[1]:
                    raise E.DimensionError(f"weight matrix must be square, got {tuple(bb.shape)}")
                if t.count_nonzero(bb - t.diag(t.diagonal(bb))).item():
                    return InnerProduct._dense(bb, host=False)
                bb = t.diagonal(bb).real.to(t.float64).contiguous()
            if bb.numel() and not bool((bb > 0).all().item()):
                raise E.NotPositiveDefinite("diagonal weight has a non-positive entry")
            return InnerProduct(kind="weighted", diag=bb)
        arr = np.asarray(b)
        if arr.ndim == 2:
            if arr.shape[0] != arr.shape[1]:
                raise E.DimensionError(f"weight matrix must be square, got {arr.shape}")
            off = arr - np.diag(np.diagonal(arr))
            if np.count_nonzero(off):
                return InnerProduct._dense(D.torch().from_numpy(np.ascontiguousarray(arr)), host=True)
            arr = np.diagonal(arr)
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        if arr.size and not np.all(arr > 0):
            raise E.NotPositiveDefinite("diagonal weight has a non-positive entry")
        return InnerProduct(kind="weighted", diag=arr)

    @property
    def n(self):
        if self.diag is not None:
            return int(self.diag.shape[0])
        return None if self.chol_b is None else int(self.chol_b.shape[0])


def _dense_basis(inner, m):
    """[L_m^{-T}; 0] = L^{-T} [I_m; 0] on the device (oblique.py:93-108)."""
    t = D.torch()
    L = inner.chol_b
    n = L.shape[0]
    dev = L.device.index
    u = t.zeros((n, m + (m & 1)), dtype=t.float64, device=L.device)
    u[:m, :m] = t.eye(m, dtype=t.float64, device=L.device)
    ctx = D.ctx(dev)
    check(lib().ots_dense_trsm_lt_f64(ctx, n, m, C.c_void_p(L.data_ptr()), n, C.c_void_p(u.data_ptr()),
                                      u.stride(0), D.stream_ptr(dev)), ctx)
    return u[:, :m]


def initial_b_basis(inner, m):
    """oblique.py:93-108 for diagonal B: [diag(d_1..m)^{-1/2}; 0] (n x m).
    Returned on the device of the weights (numpy for host weights)."""
    if inner.kind != "weighted":
        raise E.ParameterError("initial_b_basis needs a weighted inner product")
    n = inner.n
    if m > n:
        raise E.ParameterError(f"need m <= n, got m={m}, n={n}")
    if inner.diag is None:
        u = _dense_basis(inner, m)
        return u.cpu().numpy() if inner.host else u
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
    if inner.kind != "weighted":
        raise NotImplementedError("b_two_stage_qr needs a weighted inner product")
    cplx = is_complex(v) or is_complex(a)
    if inner.diag is None:
        return _b_two_stage_dense(v, a, u, inner, choice, p, n, k0, k, was_torch)
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


def _b_two_stage_dense(v, a, u, inner, choice, p, n, k0, k, was_torch):
    """Dense SPD B = L L^T with the canonical basis (module docstring)."""
    t = D.torch()
    if is_complex(v) or is_complex(a):
        raise NotImplementedError("dense complex B is not supported by this build")
    L = inner.chol_b
    dev = L.device.index
    ucan = _dense_basis(inner, k0 + k)
    ud = (u if D.is_torch(u) else t.from_numpy(np.ascontiguousarray(u))).to(device=L.device, dtype=t.float64)
    scale = float(ucan.abs().max().item()) or 1.0
    if float((ud[:, :k0 + k] - ucan).abs().max().item()) > 1e-12 * scale:
        raise NotImplementedError("this build needs u = initial_b_basis(inner, k0+k)")
    if choice not in CHOICES:
        raise E.ParameterError(f"unknown choice {choice!r}")
    ctx = D.ctx(dev)
    A = D.to_device(a, dev)
    if k0 == 0:    # b_householder_qr with the canonical basis: positive QR of L^T A, Q = L^-T Q'
        A2 = D.empty(n, k, dev)
        check(lib().ots_dense_trmm_lt_f64(ctx, n, k, C.c_void_p(L.data_ptr()), n, A.ptr, A.ld, A2.ptr, A2.ld,
                                          D.stream_ptr(dev)), ctx)
        qr = householder_qr(A2.view(), nonneg_diag=True)
        Q = D.to_device(qr.q, dev)
        check(lib().ots_dense_trsm_lt_f64(ctx, n, k, C.c_void_p(L.data_ptr()), n, Q.ptr, Q.ld,
                                          D.stream_ptr(dev)), ctx)
        z = t.zeros((0, k), dtype=t.float64, device=L.device)
        if was_torch:
            return TwoStageResult(Q.view(), qr.r, z, ReflectorDiagnostics(1.0, 0.0))
        return TwoStageResult(Q.numpy(), qr.r.cpu().numpy(), np.zeros((0, k)), ReflectorDiagnostics(1.0, 0.0))
    V = D.to_device(v, dev)
    P = D.to_device(p, dev) if (choice == "explicit" and p is not None) else None
    if choice == "explicit" and P is None:
        raise E.ParameterError("choice='explicit' requires a seed matrix p")
    Q, R, S = D.empty(n, k, dev), D.zeros(k, k, dev), D.empty(k0, k, dev)
    diag = (C.c_double * 3)()
    rc = lib().ots_b_two_stage_dense_f64(
        ctx, n, k0, k, V.ptr, V.ld, A.ptr, A.ld, C.c_void_p(L.data_ptr()), n, CHOICES[choice],
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
