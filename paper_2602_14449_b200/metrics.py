"""Stability metrics on the GPU (metrics.py:25-73 of the reference).

The reference takes exact SVDs of the n x (k0+k) block; at n = 2^24 that is
impractical, so these run Gram-based on the device:
loss = max |lambda([v?, q]^* [v?, q]) - 1|, cross = ||v^* q||_F and the
relative residual sqrt(lambda_max(E^T E) / lambda_max(A^T A)) with
E = a - v s - q r formed explicitly (never by Gram expansion).  Grams use the
DMMA tn kernel, spectra a tridiagonalisation + multisection (C-ABI
`ots_stability_f64` / `ots_stability_c128`; complex data runs on the real
views with the Grams embedded as [[Re, -Im], [Im, Re]]).  A diagonal weight
is applied as D^1/2 scaling of v and q (the cached-Cholesky path of the
reference for M = diag(d)).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _device as D
from . import errors as E
from ._native import check, lib
from .core import as_matrix, is_complex


@dataclass
class StabilityReport:
    """metrics.py:15-22."""
    loss_orth: float
    cross_orth: float
    rel_residual: float
    kappa_t: float
    scheme: str = ""
    status: str = "ok"


def _weighted(x, inner):
    if inner is None or inner.kind != "weighted":
        return x
    if inner.diag is None:       # dense B = L L^T: the B-metrics are the Euclidean ones of L^T x
        from .oblique import _phi
        return _phi(inner, x, x.device.index)
    t = D.torch()
    d = inner.diag if D.is_torch(inner.diag) else t.from_numpy(inner.diag)
    d = d.to(device=x.device, dtype=t.float64)
    return x * d.sqrt()[:, None]


def _run(v, a, q, r, s, augmented, inner=None):
    t = D.torch()
    dev = D.pick_device(q, a, v)
    raw = [x for x in (q, a, v, r, s) if x is not None]
    cplx = any(is_complex(x) for x in raw)      # decided on the raw inputs, before any cast
    dt = t.complex128 if cplx else t.float64
    to = lambda x: None if x is None else (x if D.is_torch(x) else t.from_numpy(as_matrix(x))).to(
        device=f"cuda:{dev}", dtype=dt)
    q, a, v, r, s = to(q), to(a), to(v), to(r), to(s)
    todev = D.cto_device if cplx else D.to_device
    mk = D.cempty if cplx else D.empty
    fn = lib().ots_stability_c128 if cplx else lib().ots_stability_f64
    qw = _weighted(q, inner)
    vw = _weighted(v, inner) if v is not None else None
    n, k = q.shape
    k0 = 0 if vw is None else vw.shape[1]
    Q = todev(qw.contiguous(), dev)
    V = todev(vw.contiguous(), dev) if vw is not None else None
    A = todev(a.contiguous(), dev) if a is not None else None
    R = todev(r, dev) if r is not None else None
    S = todev(s, dev) if (s is not None and k0) else None
    Eb = mk(n, k, dev)
    out = (C.c_double * 3)()
    ctx = D.ctx(dev)
    if A is not None and inner is not None and inner.kind == "weighted":
        # the residual is unweighted (a - v s - q r): use the unscaled q, v
        Q2 = todev(q.contiguous(), dev)
        V2 = todev(v.contiguous(), dev) if v is not None else None
        rc = fn(ctx, n, k0, k, V2.ptr if V2 else None, V2.ld if V2 else 0, A.ptr, A.ld,
                Q2.ptr, Q2.ld, R.ptr, R.ld, S.ptr if S else None, S.ld if S else 0,
                0, Eb.ptr, Eb.ld, out, D.stream_ptr(dev))
        check(rc, ctx)
        resid = out[2]
        rc = fn(ctx, n, k0, k, V.ptr if V else None, V.ld if V else 0, None, 0,
                Q.ptr, Q.ld, None, 0, None, 0, 1 if augmented else 0, Eb.ptr, Eb.ld,
                out, D.stream_ptr(dev))
        check(rc, ctx)
        return float(out[0]), float(out[1]), float(resid)
    rc = fn(ctx, n, k0, k, V.ptr if V else None, V.ld if V else 0,
            A.ptr if A else None, A.ld if A else 0, Q.ptr, Q.ld,
            R.ptr if R else None, R.ld if R else 0, S.ptr if S else None,
            S.ld if S else 0, 1 if augmented else 0, Eb.ptr, Eb.ld, out,
            D.stream_ptr(dev))
    check(rc, ctx)
    return float(out[0]), float(out[1]), float(out[2])


def orthogonality_loss(q, inner=None, v=None):
    """metrics.py:25-39: ||q^* B q - I||_2, or the [v, q]-augmented variant."""
    if q.shape[0] == 0 or q.shape[1] == 0:
        return 0.0
    loss, _, _ = _run(v, None, q, None, None, augmented=v is not None, inner=inner)
    return loss


def compute_metrics(v, a, result, inner=None, augmented=False, scheme=""):
    """metrics.py:42-68."""
    q = result.q
    if v is not None and v.shape[0] != q.shape[0]:
        raise E.DimensionError("v and q must share the row count")
    if a.shape[0] != q.shape[0]:
        raise E.DimensionError("a and q must share the row count")
    s = getattr(result, "s", None)
    loss, cross, resid = _run(v, a, q, result.r, s, augmented, inner)
    if v is None or v.shape[1] == 0:
        cross = 0.0
    diag = getattr(result, "diagnostics", None)
    kappa_t = diag.kappa_t if diag is not None else float("nan")
    return StabilityReport(loss_orth=loss, cross_orth=cross, rel_residual=resid, kappa_t=kappa_t,
                           scheme=scheme)


def failed_report(scheme=""):
    """metrics.py:71-75."""
    nan = float("nan")
    return StabilityReport(loss_orth=nan, cross_orth=nan, rel_residual=nan, kappa_t=nan, scheme=scheme,
                           status="intra_failed")
