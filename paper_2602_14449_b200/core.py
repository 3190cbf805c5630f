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


def _qr_signs(qtop):
    """LAPACK sign vector (device tensor, +-1) of a positive-diagonal QR from
    its Q's top k x k block (ots_qr_signs_*)."""
    t = D.torch()
    k = qtop.shape[0]
    dev = qtop.device.index
    ctx = D.ctx(dev)
    svec = t.empty(max(k, 1), dtype=t.float64, device=qtop.device)
    if is_complex(qtop):
        Qt = D.cto_device(qtop, dev)
        rc = lib().ots_qr_signs_c128(ctx, k, Qt.ptr, Qt.ld, C.c_void_p(svec.data_ptr()), D.stream_ptr(dev))
    else:
        Qt = D.to_device(qtop, dev)
        rc = lib().ots_qr_signs_f64(ctx, k, Qt.ptr, Qt.ld, C.c_void_p(svec.data_ptr()), D.stream_ptr(dev))
    check(rc, ctx)
    return svec[:k]


def _householder_qr_wide(a, nonneg_diag, was_torch):
    """k > 64 columns: Algorithm 3 over 64-column blocks on the device (block
    0 by the TSQR, block i by Algorithm 1 against the accumulated Q), then
    the LAPACK sign convention of the whole matrix recovered from Q's top
    k x k block (the QR with positive diagonal is unique, and the
    modified-LU rule on its Q gives dgeqrf's signs).  Same Q, R as LAPACK on
    full-rank input up to rounding."""
    from .twostage import block_householder_qr
    t = D.torch()
    m, n = a.shape
    dev = D.pick_device(a)
    dt = t.complex128 if is_complex(a) else t.float64
    ad = (a if D.is_torch(a) else t.from_numpy(a)).to(device=f"cuda:{dev}", dtype=dt)
    res = block_householder_qr([ad[:, c:c + 64] for c in range(0, n, 64)])
    q, r = res.q, res.r
    dg = t.diagonal(r).real
    d = t.where(dg < 0, -1.0, 1.0).to(t.float64)
    q = q * d.to(dt)[None, :]
    r = r * d.to(dt)[:, None]
    s = _qr_signs(q[:n, :n]).to(dt)
    q = (q * s[None, :]).contiguous()
    r = t.triu(r * s[:, None])
    if nonneg_diag:
        ph = t.where(t.diagonal(r).real < 0, -1.0, 1.0).to(dt)
        q = q * ph[None, :]
        r = r * ph[:, None]
    if not t.isfinite(r).all():
        raise ValueError("input contains non-finite entries")
    return QRPair(q if was_torch else q.cpu().numpy(), r if was_torch else r.cpu().numpy())


def householder_qr(a, nonneg_diag=False):
    """QR of a tall matrix on the GPU (core.py:61-84 semantics)."""
    was_torch = D.is_torch(a)
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise E.DimensionError(f"need rows >= cols, got {m}x{n}")
    if n > 64:
        return _householder_qr_wide(a, nonneg_diag, was_torch)
    # non-finite input: ValueError from the device (R check, core.py:72-73)
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


def _shifted_cholesky_qr_wide(a, refine_passes, was_torch):
    """k > 64: the same algorithm (core.py:177-202) with the n-length Grams
    and updates on the device kernels (ots_gram_* / ots_update_*) and the
    k x k shift / Cholesky / triangular inverse as small device ops."""
    from .oblique import _tcholesky
    t = D.torch()
    m, n = a.shape
    dev = D.pick_device(a)
    dt = t.complex128 if is_complex(a) else t.float64
    x = (a if D.is_torch(a) else t.from_numpy(a)).to(device=f"cuda:{dev}", dtype=dt)

    def inv_h(l):
        return t.linalg.solve_triangular(l, t.eye(n, dtype=l.dtype, device=l.device), upper=False).mH

    g = gram(x)
    g = (g + g.mH) / 2.0
    shift = 11.0 * (m * n + n * (n + 1)) * EPS * spectral_norm(g)     # ||g||_2 from the device spectrum
    l = _tcholesky(g + shift * t.eye(n, dtype=g.dtype, device=g.device))
    q = update(x, inv_h(l))
    r = l.mH
    for _ in range(refine_passes):
        g2 = gram(q)
        g2 = (g2 + g2.mH) / 2.0
        l2 = _tcholesky(g2)
        q = update(q, inv_h(l2))
        r = l2.mH @ r
    r = t.triu(r)
    return QRPair(q if was_torch else q.cpu().numpy(), r if was_torch else r.cpu().numpy())


def shifted_cholesky_qr(a, refine_passes=2):
    """Shifted Cholesky-QR + `refine_passes` unshifted refinements on the GPU
    (core.py:177-202).  Breakdown raises NotPositiveDefinite."""
    refine_passes = max(0, int(refine_passes))
    was_torch = D.is_torch(a)
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise E.DimensionError(f"need rows >= cols, got {m}x{n}")
    if n > 64:
        return _shifted_cholesky_qr_wide(a, refine_passes, was_torch)
    dev = D.pick_device(a)
    ctx = D.ctx(dev)
    if is_complex(a):
        A = D.cto_device(a, dev)
        Q = D.cempty(m, n, dev)
        R = D.czeros(n, n, dev)
        if n:
            rc = lib().ots_shifted_cholesky_qr_ex_c128(ctx, m, n, A.ptr, A.ld, Q.ptr, Q.ld, R.ptr, R.ld,
                                                       refine_passes, D.stream_ptr(dev))
            check(rc, ctx)
        return QRPair(out_like(was_torch, Q), out_like(was_torch, R))
    A = D.to_device(a, dev)
    Q = D.empty(m, n, dev)
    R = D.zeros(n, n, dev)
    if n:
        rc = lib().ots_shifted_cholesky_qr_ex_f64(ctx, m, n, A.ptr, A.ld, Q.ptr, Q.ld, R.ptr, R.ld,
                                                  refine_passes, D.stream_ptr(dev))
        check(rc, ctx)
    return QRPair(out_like(was_torch, Q), out_like(was_torch, R))


# ---------------------------------------------------------------------------
# n-length block products on the device (DMMA kernels of the path), used by
# the drivers, the comparators (baselines.py) and the weighted inner product
# ---------------------------------------------------------------------------
def _dev_of(*xs):
    return D.pick_device(*xs)


def _tdev(x, dev, cplx):
    t = D.torch()
    dt = t.complex128 if cplx else t.float64
    x = x if D.is_torch(x) else t.from_numpy(np.ascontiguousarray(x))
    return x.to(device=f"cuda:{dev}", dtype=dt)


def gram(p, b=None):
    """p^* b (p n x q1, b n x q2) on the GPU -> CUDA tensor (q1 x q2);
    b None: the Hermitian p^* p."""
    t = D.torch()
    cplx = is_complex(p) or (b is not None and is_complex(b))
    dev = _dev_of(p, b) if b is not None else _dev_of(p)
    todev = D.cto_device if cplx else D.to_device
    P = todev(_tdev(p, dev, cplx), dev)
    B = todev(_tdev(b, dev, cplx), dev) if b is not None else None
    q = P.cols if B is None else B.cols
    out = t.empty((max(P.cols, 1), max(q, 1)), dtype=t.complex128 if cplx else t.float64, device=f"cuda:{dev}")
    ctx = D.ctx(dev)
    fn = lib().ots_gram_c128 if cplx else lib().ots_gram_f64
    rc = fn(ctx, P.rows if p.shape[0] else 0, P.cols, P.ptr, P.ld, q, B.ptr if B is not None else None,
            B.ld if B is not None else 0, C.c_void_p(out.data_ptr()), out.stride(0), D.stream_ptr(dev))
    check(rc, ctx)
    return out[:P.cols, :q]


def update(v, z, b=None):
    """b + v z (v n x p, z p x m, b n x m or None) on the GPU -> CUDA tensor."""
    cplx = is_complex(v) or is_complex(z) or (b is not None and is_complex(b))
    dev = _dev_of(v, z, b) if b is not None else _dev_of(v, z)
    todev = D.cto_device if cplx else D.to_device
    V = todev(_tdev(v, dev, cplx), dev)
    Z = todev(_tdev(z, dev, cplx), dev)
    B = todev(_tdev(b, dev, cplx), dev) if b is not None else None
    n, m = v.shape[0], z.shape[1]
    X = (D.cempty if cplx else D.empty)(n, m, dev)
    ctx = D.ctx(dev)
    fn = lib().ots_update_c128 if cplx else lib().ots_update_f64
    rc = fn(ctx, n, V.cols, V.ptr, V.ld, m, Z.ptr, Z.ld, B.ptr if B is not None else None,
            B.ld if B is not None else 0, X.ptr, X.ld, D.stream_ptr(dev))
    check(rc, ctx)
    return X.view()[:n]


def gram_extremes(v):
    """(lambda_min, lambda_max) of v^* v from the device Gram + spectrum."""
    if v.shape[1] == 0:
        return 0.0, 0.0
    v = as_matrix(v, "v")
    dev = D.pick_device(v)
    ctx = D.ctx(dev)
    out = (C.c_double * 2)()
    if is_complex(v):
        V = D.cto_device(v, dev)
        rc = lib().ots_gram_extremes_c128(ctx, v.shape[0], V.cols, V.ptr, V.ld, out, D.stream_ptr(dev))
    else:
        V = D.to_device(v, dev)
        rc = lib().ots_gram_extremes_f64(ctx, v.shape[0], V.cols, V.ptr, V.ld, out, D.stream_ptr(dev))
    check(rc, ctx)
    return float(out[0]), float(out[1])


def spectral_norm(a):
    """||a||_2 (core.py:35-40) = sqrt(lambda_max(a^* a)) on the GPU (for the
    tall blocks of this path; the reference takes an SVD)."""
    if a.shape[0] == 0 or a.shape[1] == 0:
        return 0.0
    return float(np.sqrt(max(gram_extremes(a)[1], 0.0)))


def orthonormality_defect(v):
    """||v^* v - I||_2 (core.py:43-49) on the GPU: DMMA Gram + symmetric
    spectrum (ots_orthonormality_defect_*)."""
    was_torch = D.is_torch(v)
    if not was_torch:
        v = np.asarray(v)
    if v.shape[0] == 0 or v.shape[1] == 0:
        return 0.0
    v = as_matrix(v, "v")
    dev = D.pick_device(v)
    ctx = D.ctx(dev)
    out = C.c_double()
    if is_complex(v):
        V = D.cto_device(v, dev)
        rc = lib().ots_orthonormality_defect_c128(ctx, v.shape[0], V.cols, V.ptr, V.ld, C.byref(out),
                                                  D.stream_ptr(dev))
    else:
        V = D.to_device(v, dev)
        rc = lib().ots_orthonormality_defect_f64(ctx, v.shape[0], V.cols, V.ptr, V.ld, C.byref(out),
                                                 D.stream_ptr(dev))
    check(rc, ctx)
    return float(out.value)
