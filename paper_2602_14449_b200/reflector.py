"""Generalized Householder reflector API (reflector.py of the reference).

The reflector H = I - W T^{-1} W^* is constructed on the GPU from the k0 x k0
top block of V (seed kernels in csrc/small.cu).  In this build the
reflector objects are produced and consumed inside `two_stage_qr`; the
standalone pieces exposed here are `modified_lu` (Algorithm 2) and the
record types."""

from __future__ import annotations

import ctypes as C
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


class _DeviceTSolver:
    """T-solver of a device reflector (reflector.py:80-153): solve(b, adjoint)
    and reconstruct() run on the GPU."""

    kinds = {"mlu": "mlu", "qr": "tri", "polar": "chol", "explicit": "lu"}

    def __init__(self, handle, choice, k0, dev, like_torch):
        self._h, self.kind, self.k0, self._dev, self._torch = handle, self.kinds[choice], k0, dev, like_torch

    def solve(self, b, adjoint=False):
        was_torch = D.is_torch(b)
        if self._h.cplx:    # complex T: pivoted LU of phi(T) on the device
            bb = as_matrix(b if (was_torch or np.ndim(b) == 2) else np.asarray(b)[:, None], "b")
            vec = (not was_torch) and np.ndim(b) == 1
            out = D.cto_device(bb, self._dev)
            out = D.DMat(out.buf.clone(), out.cols, ld=out.ld) if was_torch else out
            ctx = D.ctx(self._dev)
            check(lib().ots_reflector_tsolve_c128(ctx, self._h.ptr, out.cols, out.ptr, out.ld, int(bool(adjoint)),
                                                  D.stream_ptr(self._dev)), ctx)
            res = out.view() if was_torch else out.numpy()
            return res[:, 0] if vec else res
        if is_complex(b):   # T is real: real and imaginary parts separately
            re = self.solve(b.real.contiguous() if was_torch else np.ascontiguousarray(np.real(b)), adjoint)
            im = self.solve(b.imag.contiguous() if was_torch else np.ascontiguousarray(np.imag(b)), adjoint)
            return D.torch().complex(re, im) if was_torch else re + 1j * im
        bb = as_matrix(b if (was_torch or np.ndim(b) == 2) else np.asarray(b)[:, None], "b")
        vec = (not was_torch) and np.ndim(b) == 1
        B = D.to_device(bb, self._dev)
        out = D.empty(B.rows, B.cols, self._dev)
        out.buf[:, :B.cols].copy_(B.view())
        ctx = D.ctx(self._dev)
        check(lib().ots_reflector_tsolve_f64(ctx, self._h.ptr, B.cols, out.ptr, out.ld, int(bool(adjoint)),
                                             D.stream_ptr(self._dev)), ctx)
        res = out.view() if was_torch else out.numpy()
        return res[:, 0] if vec else res

    def reconstruct(self):
        return self._h.get(1, self._torch)


class _Handle:
    def __init__(self, ptr, dev, cplx=False):
        import weakref
        self.ptr = ptr
        self.dev = dev
        self.cplx = cplx
        destroy = lib().ots_zreflector_destroy if cplx else lib().ots_reflector_destroy
        self._fin = weakref.finalize(self, destroy, ptr)

    def get(self, which, as_torch):
        ctx = D.ctx(self.dev)
        k0 = self.k0
        out = (D.cempty if self.cplx else D.empty)(k0, k0, self.dev)
        fn = lib().ots_reflector_get_c128 if self.cplx else lib().ots_reflector_get_f64
        check(fn(ctx, self.ptr, which, out.ptr, out.ld, D.stream_ptr(self.dev)), ctx)
        return out.view().clone() if as_torch else out.numpy()


class GenHouseholder:
    """reflector.py:156-165.  Device-backed: `w` is materialised lazily
    (W = -V with the top k0 rows replaced by fl(P - V_t)), `p` and
    `t_solver` read the seed state from the device."""

    def __init__(self, handle, V, choice, n, k0, like_torch):
        self._h, self._V, self.choice, self.n, self.k0 = handle, V, choice, n, k0
        self._torch = like_torch
        handle.k0 = k0
        self.t_solver = _DeviceTSolver(handle, choice, k0, handle.dev, like_torch)
        self._w = None

    @property
    def p(self):
        return self._h.get(0, self._torch)

    @property
    def w(self):
        if self._w is None:
            t = D.torch()
            V = self._V.view()
            w = -V.clone()
            p = t.as_tensor(self.p, device=V.device) if not self._torch else self.p
            p = p.to(w.dtype)
            w[:self.k0] = p - V[:self.k0]
            self._w = w if self._torch else w.cpu().numpy()
        return self._w


def build_reflector(v, choice="qr", p=None, orth_tol=1e-8, allow_defect=False):
    """reflector.py:207-228 on the GPU (defect check, seed, W_top)."""
    import ctypes as C
    was_torch = D.is_torch(v)
    v = as_matrix(v, "v")
    n, k0 = v.shape
    if k0 > n:
        raise E.DimensionError(f"v must be tall, got {tuple(v.shape)}")
    if k0 == 0:
        raise E.DimensionError("v must have at least one column")
    cplx = is_complex(v)

    def deferred(exc):   # the defect check (reflector.py:220-223) precedes the seed's checks
        if not allow_defect:
            from .core import orthonormality_defect
            defect = orthonormality_defect(v)
            if defect > orth_tol:
                raise E.OrthonormalityError(f"||v^* v - I||_2 = {defect:.3e} exceeds {orth_tol:.1e}")
        raise exc

    if choice not in CHOICES:
        deferred(E.ParameterError(f"unknown choice {choice!r}; expected one of {CHOICES}"))
    dev = D.pick_device(v)
    ctx = D.ctx(dev)
    todev = D.cto_device if cplx else D.to_device
    V = todev(v, dev)
    P = None
    if choice == "explicit":
        if p is None:
            deferred(E.ParameterError("choice='explicit' requires a seed matrix p"))
        try:
            p = as_matrix(p, "p")
        except E.DimensionError as exc:
            deferred(exc)
        if tuple(p.shape) != (k0, k0):
            deferred(E.DimensionError(f"seed p must be {k0}x{k0}, got {tuple(p.shape)}"))
        P = todev(p, dev)
    h = C.c_void_p()
    defect = C.c_double()
    from ._native import CHOICES as _CH
    fn = lib().ots_build_reflector_c128 if cplx else lib().ots_build_reflector_f64
    rc = fn(ctx, n, k0, V.ptr, V.ld, _CH[choice], P.ptr if P is not None else None, P.ld if P is not None else 0,
            orth_tol, int(bool(allow_defect)), C.byref(h), C.byref(defect), D.stream_ptr(dev))
    check(rc, ctx)
    return GenHouseholder(_Handle(h, dev, cplx), V, choice, n, k0, was_torch)


def apply_reflector(h, x, adjoint=False):
    """reflector.py:231-238: x - W T^{-(*)} (W^* x), on the GPU."""
    was_torch = D.is_torch(x)
    x = as_matrix(x, "x")
    if x.shape[0] != h.n:
        raise E.DimensionError(f"x has {x.shape[0]} rows, reflector expects {h.n}")
    cplx = h._h.cplx
    if is_complex(x) and not cplx:   # a real reflector acts on the real and imaginary parts separately
        re = apply_reflector(h, x.real.contiguous() if was_torch else np.ascontiguousarray(x.real), adjoint)
        im = apply_reflector(h, x.imag.contiguous() if was_torch else np.ascontiguousarray(x.imag), adjoint)
        return D.torch().complex(re, im) if was_torch else re + 1j * im
    dev = h._h.dev
    ctx = D.ctx(dev)
    todev, mk = (D.cto_device, D.cempty) if cplx else (D.to_device, D.empty)
    fn = lib().ots_apply_reflector_c128 if cplx else lib().ots_apply_reflector_f64
    X = todev(x, dev)
    m = X.cols
    Y = mk(h.n, m, dev)
    esz = 16 if cplx else 8
    for c0 in range(0, m, 64):      # 64 columns per call; column views, no copies
        c1 = min(m, c0 + 64)
        xp = C.c_void_p(X.buf.data_ptr() + c0 * esz)
        yp = C.c_void_p(Y.buf.data_ptr() + c0 * esz)
        check(fn(ctx, h._h.ptr, c1 - c0, xp, X.ld, yp, Y.ld, int(bool(adjoint)), D.stream_ptr(dev)), ctx)
    return Y.view() if was_torch else Y.numpy()


def reflector_diagnostics(h):
    """reflector.py:241-247 from k0 x k0 device data."""
    import ctypes as C
    ctx = D.ctx(h._h.dev)
    d = (C.c_double * 2)()
    fn = lib().ots_reflector_diagnostics_c128 if h._h.cplx else lib().ots_reflector_diagnostics_f64
    check(fn(ctx, h._h.ptr, d, D.stream_ptr(h._h.dev)), ctx)
    return ReflectorDiagnostics(float(d[0]), float(d[1]))


def modified_lu(z):
    """Pivot-free LU of diag(p) - z with on-the-fly signs (reflector.py:53-77,
    PAPER Alg. 2), on the GPU.  NormBoundError if ||z||_2 > 1 + 1e-8."""
    was_torch = D.is_torch(z)
    z = as_matrix(z, "z")
    k = z.shape[0]
    if z.shape[0] != z.shape[1]:
        raise E.DimensionError(f"modified_lu needs a square matrix, got {tuple(z.shape)}")
    cplx = is_complex(z)
    if k == 0:
        e = np.zeros((0, 0), dtype=np.complex128 if cplx else np.float64)
        return MLUResult(np.ones(0), e, e)
    dev = D.pick_device(z)
    ctx = D.ctx(dev)
    Z = (D.cto_device if cplx else D.to_device)(z, dev)
    t = D.torch()
    dt = t.complex128 if cplx else t.float64
    LU = t.empty((k, k), dtype=dt, device=f"cuda:{dev}")
    p = t.empty((k,), dtype=t.float64, device=f"cuda:{dev}")
    import ctypes as C
    fn = lib().ots_modified_lu_c128 if cplx else lib().ots_modified_lu_f64
    rc = fn(ctx, k, Z.ptr, Z.ld, C.c_void_p(LU.data_ptr()), C.c_void_p(p.data_ptr()), D.stream_ptr(dev))
    check(rc, ctx)
    lo = t.tril(LU, -1) + t.eye(k, dtype=dt, device=LU.device)
    up = t.triu(LU)
    if was_torch:
        return MLUResult(p, lo, up)
    return MLUResult(p.cpu().numpy(), lo.cpu().numpy(), up.cpu().numpy())
