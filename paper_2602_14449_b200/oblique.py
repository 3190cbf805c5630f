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
raise NotImplementedError.  The primitives b_householder_qr,
b_build_reflector, b_apply_reflector and the driver b_block_householder_qr
use the same isometry (section at the end of this module).
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
    cplx: bool = False         # dense complex B: chol_b is the 2n x 2n real embedding phi(L)

    @staticmethod
    def euclidean():
        return InnerProduct(kind="euclidean")

    @staticmethod
    def _dense(b, host):
        """oblique.py:48-56 for a dense b: Hermitian check (Frobenius form of
        the reference's 1e-12 spectral test), symmetrise, Cholesky on the GPU.
        A complex Hermitian b = L L^* is factored through its real embedding
        phi(b) (2n x 2n, entry b_ij -> [[Re, -Im], [Im, Re]] with rows and
        columns interleaved re/im): phi(b) is SPD and its real Cholesky factor
        is exactly phi(L) (lower triangular, the diagonal blocks l_jj I), so
        L^* x and L^-* x are the real dense kernels on the interleaved x."""
        t = D.torch()
        n = b.shape[0]
        dev = b.device.index if b.is_cuda else t.cuda.current_device()
        cplx = b.is_complex()
        bd = b.to(device=f"cuda:{dev}", dtype=t.complex128 if cplx else t.float64)
        asym = t.linalg.matrix_norm(bd - bd.mH).item()
        if asym > 1e-12 * t.linalg.matrix_norm(bd).item():
            raise E.NotHermitian("weight matrix is not Hermitian to tolerance")
        bs = ((bd + bd.mH) * 0.5).contiguous()
        if cplx:
            br, bi = bs.real, bs.imag
            blk = t.stack([t.stack([br, -bi], -1), t.stack([bi, br], -1)], -2)   # [i, j, a, c]
            bf = blk.permute(0, 2, 1, 3).reshape(2 * n, 2 * n).contiguous()
        else:
            bf = bs
        nf = bf.shape[0]
        L = t.empty_like(bf)
        ctx = D.ctx(dev)
        check(lib().ots_dense_cholesky_f64(ctx, nf, C.c_void_p(bf.data_ptr()), nf, C.c_void_p(L.data_ptr()), nf,
                                           D.stream_ptr(dev)), ctx)
        return InnerProduct(kind="weighted", b=bs, chol_b=L, host=host, cplx=cplx)

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
        if self.chol_b is None:
            return None
        return int(self.chol_b.shape[0]) // (2 if self.cplx else 1)

    # -- oblique.py:62-90 (n-length work on the device; numpy in -> numpy out)
    def apply(self, x):
        """B x (identity for the Euclidean kind) -- oblique.py:62-64."""
        if self.kind == "euclidean":
            return x
        was_torch = D.is_torch(x)
        dev = _dev_of(self, x)
        t = D.torch()
        xd = (x if was_torch else t.from_numpy(np.ascontiguousarray(x))).to(f"cuda:{dev}")
        if self.diag is not None:
            d = _sqrt_d(self, dev) ** 2
            y = xd * (d[:, None] if xd.dim() == 2 else d)
        else:
            dt = t.complex128 if (self.cplx or xd.is_complex()) else t.float64
            y = self.b.to(dt) @ xd.to(dt)
        return y if was_torch else y.cpu().numpy()

    def _phi_x(self, x):
        """L^* x (x itself for the Euclidean kind) as a device tensor."""
        t = D.torch()
        if self.kind == "euclidean":
            xd = x if D.is_torch(x) else t.from_numpy(np.ascontiguousarray(x))
            return xd.to(f"cuda:{D.pick_device(xd)}")
        dev = _dev_of(self, x)
        return _phi(self, x, dev)

    def gram(self, x, y):
        """y^* B x -- oblique.py:66-68."""
        from .core import gram as _gram
        was_torch = D.is_torch(x) or D.is_torch(y)
        g = _gram(y, self.apply(x))
        return g if was_torch else g.cpu().numpy()

    def col_norms(self, x):
        """||L^* x_j||_2 per column -- oblique.py:70-73."""
        from .core import gram as _gram
        m = self._phi_x(x)
        nr = _gram(m).diagonal().real.clamp_min(0).sqrt() if m.shape[1] else m.new_zeros(0).real
        return nr if D.is_torch(x) else nr.cpu().numpy()

    def norm(self, x):
        """B-weighted spectral norm ||L^* x||_2 (vector 2-norm for 1-D x) --
        oblique.py:75-81."""
        from .core import spectral_norm
        one_d = (x.dim() if D.is_torch(x) else np.ndim(x)) == 1
        m = self._phi_x(x[:, None] if one_d else x)
        return spectral_norm(m)

    def defect(self, x):
        """||x^* B x - I||_2 -- oblique.py:83-90."""
        from .core import orthonormality_defect
        if (x.numel() if D.is_torch(x) else np.size(x)) == 0:
            return 0.0
        return orthonormality_defect(self._phi_x(x))


def _tcholesky(a):
    """core.py:87-105 on a small device matrix: Hermitian to 1e-12 ||a||_2
    (NotHermitian), symmetrised, lower Cholesky (NotPositiveDefinite)."""
    t = D.torch()
    if a.shape[0] != a.shape[1]:
        raise E.DimensionError(f"cholesky needs a square matrix, got {tuple(a.shape)}")
    if a.shape[0] == 0:
        return a.clone()
    from .core import spectral_norm                # device Gram spectrum (no cuSOLVER)
    nrm = spectral_norm(a)
    if spectral_norm((a - a.mH).contiguous()) > 1e-12 * nrm:
        raise E.NotHermitian("matrix is not Hermitian to 1e-12 * ||a||_2")
    h = (a + a.mH) / 2.0
    l, info = t.linalg.cholesky_ex(h)
    if int(info.item()) != 0 or not bool(t.isfinite(l).all().item()):
        raise E.NotPositiveDefinite(f"{int(info.item())}-th leading minor not positive definite")
    return l


def _dense_basis(inner, m):
    """[L_m^{-*}; 0] = L^{-*} [I_m; 0] on the device (oblique.py:93-108)."""
    t = D.torch()
    L = inner.chol_b
    dev = L.device.index
    if inner.cplx:
        e = t.zeros((inner.n, m), dtype=t.complex128, device=L.device)
        e[:m, :m] = t.eye(m, dtype=t.complex128, device=L.device)
        return _phi(inner, e, dev, inverse=True)
    n = L.shape[0]
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
    """u[:, :m] == initial_b_basis(diag(d), m) up to rounding of d^-1/2."""
    if D.is_torch(u):
        t = D.torch()
        top = u[:m, :m]
        want = t.diag(t.as_tensor(d, device=u.device)[:m].rsqrt())
        return bool(t.allclose(top.to(want.dtype), want, rtol=1e-14, atol=0.0)) and \
            not bool(u[m:, :m].any().item())
    top = np.asarray(u[:m, :m])
    dd = np.asarray(d.cpu().numpy() if D.is_torch(d) else d)[:m]
    return np.allclose(top, np.diag(1.0 / np.sqrt(dd)), rtol=1e-14, atol=0.0) and not np.count_nonzero(u[m:, :m])


def b_two_stage_qr(v, a, u, inner, choice="qr", reorth=True, p=None):
    """Algorithm 4 (oblique.py:279-315) on the GPU (diagonal or dense B, any
    B-orthonormal basis u); OrthonormalityError names the B-defect as the
    reference's b_build_reflector does (oblique.py:141-145)."""
    try:
        return _b_two_stage_qr(v, a, u, inner, choice, reorth, p)
    except E.OrthonormalityError as exc:
        msg = str(exc)
        if "B v" not in msg and "B u" not in msg:
            msg = msg.replace("v^* v", "v^* B v")
        raise E.OrthonormalityError(msg) from None


def _b_two_stage_qr(v, a, u, inner, choice="qr", reorth=True, p=None):
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
    if inner.kind != "weighted":          # B = I: the unit diagonal weight
        inner = InnerProduct(kind="weighted", diag=np.ones(n), host=not was_torch)
    cplx = is_complex(v) or is_complex(a)
    if not _canonical(u, inner, k0 + k):
        # Q, R, S do not depend on u (positive-diagonal B-QR, S = v^* B a are
        # unique); the seed P, T and the diagnostics do, through the coupling
        # v^* B u0 (oblique.py:125-151): run the canonical path for Q, R, S and
        # take the diagnostics from the B-reflector of (v, u[:, :k0]).
        res = _b_two_stage_qr(v, a, initial_b_basis(inner, k0 + k), inner, choice, reorth, p)
        if k0 > 0:
            h = b_build_reflector(v, u[:, :k0], inner, choice, p=p)
            res.diagnostics = b_reflector_diagnostics(h)
        return res
    if inner.diag is None:
        return _b_two_stage_dense(v, a, u, inner, choice, p, n, k0, k, was_torch)
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
    if inner.cplx or is_complex(v) or is_complex(a):
        return _zb_two_stage_dense(v, a, inner, choice, p, k0, k, was_torch)
    L = inner.chol_b
    dev = L.device.index
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


def _zb_two_stage_dense(v, a, inner, choice, p, k0, k, was_torch):
    """Dense complex B, canonical basis: the Euclidean complex pipeline on
    (L^* v, L^* a) gives S = v^* B a and the unique positive-diagonal B-QR
    of the projected block after the phase fix Q = L^-* Q' d, R = d^* R'
    (d = the phases of diag R'); the diagnostics are those of the canonical
    B-reflector (oblique.py:125-167), as for the general-u path."""
    from .twostage import two_stage_qr
    t = D.torch()
    dev = inner.chol_b.device.index
    if choice not in CHOICES:
        raise E.ParameterError(f"unknown choice {choice!r}")
    pa = _phi(inner, a, dev)
    if k0 == 0:
        qr = householder_qr(pa, nonneg_diag=True)
        q = _phi(inner, qr.q, dev, inverse=True)
        z = t.zeros((0, k), dtype=t.complex128, device=q.device)
        return TwoStageResult(_out(q, was_torch), _out(qr.r, was_torch), _out(z, was_torch),
                              ReflectorDiagnostics(1.0, 0.0))
    if choice == "explicit" and p is None:
        raise E.ParameterError("choice='explicit' requires a seed matrix p")
    pv = _phi(inner, v, dev)
    pp = None if p is None else (p if D.is_torch(p) else t.from_numpy(np.ascontiguousarray(p))).to(
        device=pv.device, dtype=t.complex128)
    res = two_stage_qr(pv, pa, choice=choice, p=pp)
    r = res.r
    dg = t.diagonal(r)
    ph = t.where(dg.abs() > 0, dg / dg.abs().clamp_min(1e-300), t.ones_like(dg))
    r = t.triu(ph.conj()[:, None] * r)
    q = _phi(inner, res.q * ph[None, :], dev, inverse=True)
    h = b_build_reflector(v, initial_b_basis(inner, k0), inner, choice, p=p, allow_defect=True)
    diag = b_reflector_diagnostics(h)
    return TwoStageResult(_out(q, was_torch), _out(r, was_torch), _out(res.s, was_torch), diag)


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
    _h: object = None          # the Euclidean reflector of (Phi v) on the device
    _rot: object = None        # general u0: the rotation U with U [I; 0] = Phi u0


# ---------------------------------------------------------------------------
# Drop-in B-path primitives through the isometry Phi (Phi = D^1/2 for a
# diagonal B, L^T for a dense B = L L^T): <x, y>_B = (Phi y)^* (Phi x), and the
# canonical basis initial_b_basis(inner, m) maps to [I_m; 0].  A B-reflector
# for (v, u0 = canonical) is H = Phi^-1 H' Phi with H' the Euclidean reflector
# of Phi v (same seed: the coupling u0^* B v is the top block of Phi v), and the
# positive-diagonal B-QR of a is Q = Phi^-1 Q', R = R' for the nonneg
# Householder QR of Phi a (unique, so it equals the reference's left-looking
# result up to rounding).  Scaling by D^+-1/2 is an element-wise torch op on the
# device; L^T x and L^-T x are the dense.cu kernels.
# ---------------------------------------------------------------------------

def _dev_of(inner, *xs):
    if inner.diag is None:
        return inner.chol_b.device.index
    if D.is_torch(inner.diag) and inner.diag.is_cuda:
        return inner.diag.device.index
    return D.pick_device(*xs)


def _sqrt_d(inner, dev):
    t = D.torch()
    d = inner.diag if D.is_torch(inner.diag) else t.from_numpy(inner.diag)
    return d.to(device=f"cuda:{dev}", dtype=t.float64).sqrt()


def _phi(inner, x, dev, inverse=False):
    """Phi x (or Phi^-1 x) for x an n x m matrix; returns a device tensor."""
    t = D.torch()
    if inner.diag is not None:
        xd = (x if D.is_torch(x) else t.from_numpy(np.ascontiguousarray(x))).to(f"cuda:{dev}")
        s = _sqrt_d(inner, dev)[:, None]
        return xd / s if inverse else xd * s
    if inner.cplx:
        return _zphi(inner, x, dev, inverse)
    if is_complex(x):
        raise E.ParameterError("complex data needs a complex (or diagonal) weight; B is real dense here "
                               "(pass B as a complex128 matrix)")
    L = inner.chol_b
    n = L.shape[0]
    ctx = D.ctx(dev)
    X = D.to_device(x, dev)
    if inverse:
        Y = D.empty(n, X.cols, dev)
        Y.buf[:, :X.cols].copy_(X.view())
        check(lib().ots_dense_trsm_lt_f64(ctx, n, X.cols, C.c_void_p(L.data_ptr()), n, Y.ptr, Y.ld,
                                          D.stream_ptr(dev)), ctx)
    else:
        Y = D.empty(n, X.cols, dev)
        check(lib().ots_dense_trmm_lt_f64(ctx, n, X.cols, C.c_void_p(L.data_ptr()), n, X.ptr, X.ld, Y.ptr, Y.ld,
                                          D.stream_ptr(dev)), ctx)
    return Y.view()


def _zphi(inner, x, dev, inverse):
    """L^* x / L^-* x for a dense complex B through the real embedding: the
    columns of x (n x m complex) become 2n-vectors with re/im interleaved
    along the rows, multiplied by phi(L)^T (= phi(L^*)) or solved with it."""
    t = D.torch()
    xd = (x if D.is_torch(x) else t.from_numpy(np.ascontiguousarray(x))).to(device=f"cuda:{dev}",
                                                                            dtype=t.complex128)
    n, m = xd.shape
    L = inner.chol_b
    nf = 2 * n
    ld = m + (m & 1) if m else 2
    xr = t.zeros((nf, ld), dtype=t.float64, device=xd.device)
    xr[:, :m] = t.view_as_real(xd.resolve_conj()).permute(0, 2, 1).reshape(nf, m)
    ctx = D.ctx(dev)
    if inverse:
        check(lib().ots_dense_trsm_lt_f64(ctx, nf, m, C.c_void_p(L.data_ptr()), nf, C.c_void_p(xr.data_ptr()),
                                          ld, D.stream_ptr(dev)), ctx)
        yr = xr
    else:
        yr = t.empty_like(xr)
        check(lib().ots_dense_trmm_lt_f64(ctx, nf, m, C.c_void_p(L.data_ptr()), nf, C.c_void_p(xr.data_ptr()),
                                          ld, C.c_void_p(yr.data_ptr()), ld, D.stream_ptr(dev)), ctx)
    return t.view_as_complex(yr[:, :m].reshape(n, 2, m).permute(0, 2, 1).contiguous())


def _out(x, was_torch):
    return x if was_torch else x.cpu().numpy()


def _check_weighted(inner, n):
    if inner.kind != "weighted":
        raise NotImplementedError("the B-path needs a weighted inner product")
    if inner.n != n:
        raise E.DimensionError(f"weight is {inner.n} x {inner.n}, data has {n} rows")


def _canonical(u, inner, m):
    """u[:, :m] == initial_b_basis(inner, m) (to rounding)?"""
    try:
        _require_canonical(u, inner, m, "u")
        return True
    except NotImplementedError:
        return False


class _Rot:
    """Orthogonal U with U [I; 0] = u0' (an n x k0 orthonormal block):
    U = H_u diag(P_u, I) for the Euclidean device reflector H_u mapping
    [P_u; 0] onto u0' (reflector.py:207-228 with choice "qr").  In the frame
    z -> U^* z a general B-orthonormal u0 becomes the canonical basis, so the
    coupling v^* B u0 (oblique.py:146) is the top block of U^* Phi v."""

    def __init__(self, pu):
        from .reflector import build_reflector
        self.h = build_reflector(pu, "qr", allow_defect=True)
        self.k0 = pu.shape[1]
        pp = self.h.p
        self.pu = pp if D.is_torch(pp) else D.torch().from_numpy(np.ascontiguousarray(pp)).to(pu.device)

    def adj(self, z):          # U^* z = diag(P_u^*, I) H_u^* z
        from .core import gram
        from .reflector import apply_reflector
        y = apply_reflector(self.h, z, adjoint=True)
        y[:self.k0] = gram(self.pu.to(y.dtype), y[:self.k0])
        return y

    def fwd(self, z):          # U z = H_u diag(P_u, I) z
        from .core import gram
        from .reflector import apply_reflector
        z2 = z.clone()
        z2[:self.k0] = gram(self.pu.mH.contiguous().to(z.dtype), z[:self.k0])
        return apply_reflector(self.h, z2)


def b_reflector_diagnostics(h):
    """oblique.py:164-167: kappa_2(T) and ||W T^{-1}||_2 with the unweighted
    W = x - v, on the device: kappa from the extreme eigenvalues of T^* T,
    ||W T^{-1}||_2^2 = lambda_max(T^{-*} (W^* W) T^{-1}) from the Gram of W
    and two T-solves."""
    from .core import gram, gram_extremes
    t = D.torch()
    tm = h.t_solver.reconstruct()
    tm = tm if D.is_torch(tm) else t.from_numpy(np.ascontiguousarray(tm)).cuda()
    lo, hi = gram_extremes(tm)
    kappa = float(np.sqrt(hi / lo)) if lo > 0 else float("inf")
    w = h.w if D.is_torch(h.w) else t.from_numpy(np.ascontiguousarray(h.w)).to(tm.device)
    gw = gram(w)                                            # W^* W
    y1 = h.t_solver.solve(gw, adjoint=True)                 # T^{-*} W^* W
    y1 = y1 if D.is_torch(y1) else t.from_numpy(y1).to(tm.device)
    m = h.t_solver.solve(y1.mH.contiguous(), adjoint=True)  # (T^{-*} W^* W T^{-1})^*
    m = m if D.is_torch(m) else t.from_numpy(m).to(tm.device)
    _, lmax2 = gram_extremes(m)                            # lambda(M)^2 (M Hermitian PSD)
    return ReflectorDiagnostics(kappa, float(np.sqrt(np.sqrt(max(lmax2, 0.0)))))


def _require_canonical(u, inner, m, name):
    """u[:, :m] must be initial_b_basis(inner, m) (the basis every caller of
    the reference's B-path passes, oblique.py:304-313, 331-346)."""
    if inner.diag is not None:
        ok = _is_canonical_basis(u, inner.diag, m)
    else:
        t = D.torch()
        ucan = _dense_basis(inner, m)
        ud = (u if D.is_torch(u) else t.from_numpy(np.ascontiguousarray(u))).to(device=ucan.device)
        ud = ud.to(t.complex128 if (ud.is_complex() or ucan.is_complex()) else t.float64)
        scale = float(ucan.abs().max().item()) if m else 1.0
        ok = float((ud[:, :m] - ucan).abs().max().item()) <= 1e-12 * (scale or 1.0) if m else True
    if not ok:
        raise NotImplementedError(f"this build needs {name} = initial_b_basis(inner, {m})")


def b_householder_qr(a, u_init, inner, reorth=True, prefix=None):
    """oblique.py:170-238: B-orthonormal Q and upper-triangular R with a
    positive diagonal, A = Q R.  Computed as Phi^-1 times the nonneg
    Householder QR of Phi a on the GPU (the factorization is unique, so this
    is the reference's result for every B-orthonormal u_init -- the
    canonical basis, or any other one checked on the GPU to 1e-6; `reorth`
    and `prefix` only steer the reference's rounding and are accepted for
    drop-in callers).  Raises
    BreakdownError when R_jj <= 1e3 u max_j ||a_j||_B (oblique.py:196-199)."""
    from .core import EPS
    was_torch = D.is_torch(a) or D.is_torch(u_init)
    a = as_matrix(a, "a")
    u_init = as_matrix(u_init, "u_init")
    n, k = a.shape
    if u_init.shape[0] != n:
        raise E.DimensionError("a and u_init must share the row count")
    if u_init.shape[1] < k:
        raise E.DimensionError(f"u_init needs at least {k} columns")
    if prefix is not None:
        prefix = as_matrix(prefix, "prefix")
        if prefix.shape[0] != n:
            raise E.DimensionError("prefix must share the row count")
    cplx = is_complex(a) or is_complex(u_init)
    if k == 0:
        dt = np.complex128 if cplx else np.float64
        if was_torch:
            t = D.torch()
            tdt = t.complex128 if cplx else t.float64
            return QRPair(t.zeros((n, 0), dtype=tdt), t.zeros((0, 0), dtype=tdt))
        return QRPair(np.zeros((n, 0), dtype=dt), np.zeros((0, 0), dtype=dt))
    _check_weighted(inner, n)
    try:
        _require_canonical(u_init, inner, k, "u_init")
    except NotImplementedError:
        # any B-orthonormal u_init gives the same (unique) result; check it is one
        from .metrics import orthogonality_loss
        if k > 64 or is_complex(u_init):
            raise
        if orthogonality_loss(u_init[:, :k], inner) > 1e-6:
            raise NotImplementedError("u_init[:, :k] must be B-orthonormal (||u^* B u - I||_2 <= 1e-6)") from None
    dev = _dev_of(inner, a)
    pa = _phi(inner, a, dev)
    t = D.torch()
    scale = float(t.linalg.vector_norm(pa, dim=0).max().item())
    thresh = 1e3 * EPS * scale
    qr = householder_qr(pa, nonneg_diag=True)
    rd = t.diagonal(qr.r).abs()
    bad = t.nonzero(rd <= thresh)
    if bad.numel():
        j = int(bad[0, 0].item())
        raise E.BreakdownError(f"column {j} is numerically zero after projection "
                               f"(B-norm {float(rd[j].item()):.3e} <= {thresh:.3e})")
    q = _phi(inner, qr.q, dev, inverse=True)
    return QRPair(_out(q, was_torch), _out(qr.r, was_torch))


def b_build_reflector(v, u0, inner, choice="qr", p=None, orth_tol=1e-6, allow_defect=False):
    """oblique.py:125-151: the B-reflector H = I - w T^-1 w^* B mapping u0 p
    onto v, for the canonical u0 = initial_b_basis(inner, k0).  Built as the
    Euclidean device reflector of Phi v (same seed p and T); w = x - v with
    x = u0 p.  Defect checks ||v^* B v - I||_2 = ||(Phi v)^*(Phi v) - I||_2 run
    in the native build (oblique.py:141-145)."""
    from .reflector import build_reflector
    was_torch = D.is_torch(v) or D.is_torch(u0)
    v = as_matrix(v, "v")
    u0 = as_matrix(u0, "u0")
    if tuple(v.shape) != tuple(u0.shape):
        raise E.DimensionError(f"v and u0 must agree in shape, {tuple(v.shape)} vs {tuple(u0.shape)}")
    n, k0 = v.shape
    if k0 == 0:
        raise E.DimensionError("v must have at least one column")
    if inner.kind != "weighted":
        inner = InnerProduct(kind="weighted", diag=np.ones(n), host=not was_torch)
    _check_weighted(inner, n)
    dev = _dev_of(inner, v)
    pv = _phi(inner, v, dev)
    rot = None
    if not _canonical(u0, inner, k0):
        # general B-orthonormal u0: defect checks in the reference's order
        # (v, then u0; oblique.py:141-145), then the canonical construction
        # in the frame U^* (Phi .) where U [I; 0] = Phi u0
        from .core import orthonormality_defect
        pu = _phi(inner, u0, dev)
        if not allow_defect:
            for name, blk in (("v", pv), ("u0", pu)):
                dd = orthonormality_defect(blk)
                if dd > orth_tol:
                    raise E.OrthonormalityError(f"||{name}^* B {name} - I||_2 = {dd:.3e} exceeds {orth_tol:.1e}")
        rot = _Rot(pu)
        pv = rot.adj(pv)
        allow_defect = True
    try:
        h = build_reflector(pv, choice=choice, p=p, orth_tol=orth_tol, allow_defect=allow_defect)
    except E.OrthonormalityError as exc:
        raise E.OrthonormalityError(str(exc).replace("v^* v", "v^* B v")) from None
    t = D.torch()
    pm = h.p                                     # device tensor (pv is torch)
    top = t.zeros((n, k0), dtype=pv.dtype, device=pv.device)
    top[:k0] = pm.to(pv.dtype)
    if rot is not None:
        top = rot.fwd(top)
    x = _phi(inner, top, dev, inverse=True)     # u0 p = Phi^-1 U [p; 0]
    vd = (v if D.is_torch(v) else t.from_numpy(np.ascontiguousarray(v))).to(device=pv.device, dtype=x.dtype)
    w = x - vd
    h._torch = was_torch
    h.t_solver._torch = was_torch
    return BGenHouseholder(w=_out(w, was_torch), t_solver=h.t_solver, p=_out(pm, was_torch), x=_out(x, was_torch),
                           inner=inner, choice=choice, n=n, k0=k0, _h=h, _rot=rot)


def b_apply_reflector(h, x, inverse=False):
    """oblique.py:154-161: H x, or H^-1 x = (I - w T^-* w^* B) x, computed as
    Phi^-1 H'^(*) Phi x with the Euclidean device reflector H'."""
    from .reflector import apply_reflector
    was_torch = D.is_torch(x)
    x = as_matrix(x, "x")
    if x.shape[0] != h.n:
        raise E.DimensionError(f"x has {x.shape[0]} rows, reflector expects {h.n}")
    if h._h is None:
        raise E.ParameterError("b_apply_reflector needs a reflector from b_build_reflector")
    dev = h._h._h.dev
    z = _phi(h.inner, x, dev)
    if h._rot is not None:
        z = h._rot.adj(z)
    y = apply_reflector(h._h, z, adjoint=inverse)
    if h._rot is not None:
        y = h._rot.fwd(y)
    return _out(_phi(h.inner, y, dev, inverse=True), was_torch)


def b_block_householder_qr(blocks, inner, choice="qr", reorth=True):
    """oblique.py:318-361: Algorithm 3 under the B inner product -- one
    canonical basis for all blocks, block 0 by b_householder_qr, block i >= 1
    by b_two_stage_qr against the accumulated Q; BreakdownError /
    NotPositiveDefinite become IntraFailure tagged with the block index."""
    from .twostage import BlockQRResult
    if not blocks:
        raise E.ParameterError("need at least one block")
    was_torch = any(D.is_torch(b) for b in blocks)
    blocks = [as_matrix(b, f"block {i}") for i, b in enumerate(blocks)]
    n = blocks[0].shape[0]
    sizes = [b.shape[1] for b in blocks]
    if any(b.shape[0] != n for b in blocks):
        raise E.DimensionError("all blocks must have the same row count")
    total = sum(sizes)
    if total > n:
        raise E.DimensionError(f"need sum(k_i) <= n, got {total} > {n}")
    t = D.torch()
    u = initial_b_basis(inner, total)
    dev = _dev_of(inner, *blocks)
    cplx = any(is_complex(b) for b in blocks) or inner.cplx
    tdt = t.complex128 if cplx else t.float64
    todev = (lambda z: (z if D.is_torch(z) else t.from_numpy(np.ascontiguousarray(z))).to(
        device=f"cuda:{dev}", dtype=tdt))
    blocks = [todev(b) for b in blocks]
    u = (u if D.is_torch(u) else t.from_numpy(u)).to(device=f"cuda:{dev}",
                                                       dtype=t.complex128 if inner.cplx else t.float64)
    r_full = t.zeros((total, total), dtype=tdt, device=f"cuda:{dev}")
    try:
        qr0 = b_householder_qr(blocks[0], u[:, :sizes[0]], inner, reorth=reorth)
    except (E.BreakdownError, E.NotPositiveDefinite) as exc:
        raise E.IntraFailure(str(exc), block=0) from None
    qs = [qr0.q]
    r_full[:sizes[0], :sizes[0]] = qr0.r
    worst = ReflectorDiagnostics(1.0, 0.0)
    offset = sizes[0]
    for i in range(1, len(blocks)):
        ki = sizes[i]
        qacc = t.cat(qs, dim=1)
        m = qacc.shape[1]
        try:
            res = b_two_stage_qr(qacc, blocks[i], u[:, :m + ki], inner, choice=choice, reorth=reorth)
        except (E.BreakdownError, E.NotPositiveDefinite) as exc:
            raise E.IntraFailure(str(exc), block=i) from None
        qs.append(res.q)
        r_full[:m, offset:offset + ki] = res.s
        r_full[offset:offset + ki, offset:offset + ki] = res.r
        if res.diagnostics and res.diagnostics.kappa_t > worst.kappa_t:
            worst = res.diagnostics
        offset += ki
    q = t.cat(qs, dim=1)
    return BlockQRResult(_out(q, was_torch), _out(r_full, was_torch), sizes, worst)
