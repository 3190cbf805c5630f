"""Algorithm 1 (two-stage Householder-QR) and its drivers -- the hot path.

`two_stage_qr` (twostage.py:57-97 of the reference) runs entirely on the GPU
through one C-ABI call (`ots_two_stage_f64`, include/ots.h); see DESIGN.md
for the kernel sequence.  Host code here only validates (same order and
exception classes as the reference), moves numpy data to/from the device and
maps status codes back to exceptions."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import errors as E
from ._native import CHOICES, INTRA, check, lib
from .core import as_matrix, householder_qr, is_complex
from .reflector import ReflectorDiagnostics

INTRA_METHODS = ("householder", "cholshift")   # twostage.py:25


@dataclass
class TwoStageResult:
    """twostage.py:28-34."""
    q: object
    r: object
    s: object
    diagnostics: ReflectorDiagnostics | None = None
    sweep_history: list = field(default_factory=list)


@dataclass
class BlockQRResult:
    """twostage.py:37-42."""
    q: object
    r: object
    block_sizes: list
    diagnostics: ReflectorDiagnostics | None = None


def intra_qr(a, intra="householder"):
    """twostage.py:45-54."""
    if intra == "householder":
        return householder_qr(a)
    if intra == "cholshift":
        from .core import shifted_cholesky_qr
        try:
            return shifted_cholesky_qr(a)
        except E.NotPositiveDefinite as exc:
            raise E.IntraFailure(f"shifted Cholesky-QR broke down: {exc}") from None
    raise E.ParameterError(f"unknown intra method {intra!r}; expected {INTRA_METHODS}")


def _zeros_like(was_torch, shape, ref=None):
    cplx = ref is not None and is_complex(ref)
    if was_torch:
        t = D.torch()
        return t.zeros(shape, dtype=t.complex128 if cplx else t.float64, device=ref.device)
    return np.zeros(shape, dtype=np.complex128 if cplx else np.float64)


def two_stage_qr(v, a, choice="qr", intra="householder", p=None):
    """Orthogonalize a against orthonormal v in two stages (Algorithm 1).

    Returns TwoStageResult(q, r, s, diagnostics) with
    [v, a] = [v, q] [[I, s], [0, r]] and [v, q]^* [v, q] = I.
    numpy in -> numpy out; CUDA tensors in -> CUDA tensors out (zero-copy).
    """
    was_torch = D.is_torch(v) or D.is_torch(a)
    v = as_matrix(v, "v")
    a = as_matrix(a, "a")
    n, k0 = v.shape
    k = a.shape[1]
    if a.shape[0] != n:
        raise E.DimensionError(f"v has {n} rows but a has {a.shape[0]}")
    if k0 + k > n:
        raise E.DimensionError(f"need k0 + k <= n, got {k0}+{k} > {n}")
    cplx = is_complex(v) or is_complex(a)
    if k0 == 0:
        qr = intra_qr(a, intra)
        return TwoStageResult(qr.q, qr.r, _zeros_like(was_torch, (0, k), a),
                              ReflectorDiagnostics(1.0, 0.0))
    if k == 0:
        ref = v if is_complex(v) else a
        return TwoStageResult(_zeros_like(was_torch, (n, 0), ref), _zeros_like(was_torch, (0, 0), ref),
                              _zeros_like(was_torch, (k0, 0), ref), ReflectorDiagnostics(1.0, 0.0))
    if choice not in CHOICES:
        raise E.ParameterError(f"unknown choice {choice!r}; expected one of "
                               f"('mlu', 'qr', 'polar', 'explicit')")
    if intra not in INTRA:
        raise E.ParameterError(f"unknown intra method {intra!r}; expected {INTRA_METHODS}")
    dev = D.pick_device(v, a)
    ctx = D.ctx(dev)
    todev = D.cto_device if cplx else D.to_device
    V = todev(v, dev)
    A = todev(a, dev)
    P = None
    if choice == "explicit":
        if p is None:
            raise E.ParameterError("choice='explicit' requires a seed matrix p")
        p = as_matrix(p, "p")
        if tuple(p.shape) != (k0, k0):
            raise E.DimensionError(f"seed p must be {k0}x{k0}, got {tuple(p.shape)}")
        P = todev(p, dev)
    if cplx:
        Q = D.cempty(n, k, dev)
        R = D.czeros(k, k, dev)
        S = D.cempty(k0, k, dev)
    else:
        Q = D.empty(n, k, dev)
        R = D.zeros(k, k, dev)
        S = D.empty(k0, k, dev)
    diag = (C.c_double * 3)()
    fn = lib().ots_two_stage_c128 if cplx else lib().ots_two_stage_f64
    rc = fn(
        ctx, n, k0, k, V.ptr, V.ld, A.ptr, A.ld, CHOICES[choice], INTRA[intra],
        P.ptr if P is not None else None, P.ld if P is not None else 0,
        1e-8, 0, Q.ptr, Q.ld, R.ptr, R.ld, S.ptr, S.ld, diag, D.stream_ptr(dev))
    check(rc, ctx)   # OrthonormalityError before the non-finite ValueError (device-side order)
    return TwoStageResult(Q.view() if was_torch else Q.numpy(),
                          R.view() if was_torch else R.numpy(),
                          S.view() if was_torch else S.numpy(),
                          ReflectorDiagnostics(float(diag[0]), float(diag[1])))


def block_householder_qr(blocks, choice="qr", intra="householder"):
    """Algorithm 3 driver (twostage.py:100-151): block 0 by the intra QR,
    block i >= 1 by `two_stage_qr` against the accumulated Q (device
    resident when the blocks are CUDA tensors)."""
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
    xp = D.torch() if was_torch else np
    if was_torch:
        t = D.torch()
        dev = D.pick_device(*blocks)
        blocks = [b if b.is_cuda else b.to(f"cuda:{dev}") for b in blocks]
        r_full = t.zeros((total, total), dtype=t.float64, device=blocks[0].device)
    else:
        r_full = np.zeros((total, total))
    try:
        qr0 = intra_qr(blocks[0], intra)
    except E.IntraFailure as exc:
        exc.block = 0
        raise
    qs = [qr0.q]
    r_full[:sizes[0], :sizes[0]] = qr0.r
    worst = ReflectorDiagnostics(1.0, 0.0)
    offset = sizes[0]
    for i in range(1, len(blocks)):
        ki = sizes[i]
        qacc = xp.hstack(qs) if not was_torch else D.torch().cat(qs, dim=1)
        try:
            res = two_stage_qr(qacc, blocks[i], choice, intra)
        except E.IntraFailure as exc:
            exc.block = i
            raise
        qs.append(res.q)
        m = qacc.shape[1]
        r_full[:m, offset:offset + ki] = res.s
        r_full[offset:offset + ki, offset:offset + ki] = res.r
        if res.diagnostics.kappa_t > worst.kappa_t:
            worst = res.diagnostics
        offset += ki
    q = D.torch().cat(qs, dim=1) if was_torch else np.hstack(qs)
    return BlockQRResult(q, r_full, sizes, worst)


def reorthogonalized_two_stage(v, a, choice="qr", intra="householder", sweeps=1, sequence=None):
    """twostage.py:154-180 for choice != 'bcgs' (repeated Algorithm-1 passes)."""
    if choice == "bcgs":
        raise NotImplementedError("BCGS baselines are out of scope for the GPU path")
    if sweeps < 1:
        raise E.ParameterError("sweeps must be >= 1")
    res = two_stage_qr(v, a, choice, intra)
    history = [_augmented_defect(v, res.q)]
    q, r, s = res.q, res.r, res.s
    diag = res.diagnostics
    for _ in range(sweeps - 1):
        nxt = two_stage_qr(v, q, choice, intra)
        s = s + nxt.s @ r
        r = nxt.r @ r
        q = nxt.q
        diag = nxt.diagnostics
        history.append(_augmented_defect(v, q))
    return TwoStageResult(q, r, s, diag, sweep_history=history)


def _augmented_defect(v, q):
    """||[v, q]^*[v, q] - I||_2 from the (k0+k)^2 Gram (host eigvalsh on the
    small Gram; the n-length Gram itself is formed on the device when the
    inputs are CUDA tensors)."""
    if D.is_torch(q):
        t = D.torch()
        vq = t.cat([v.to(q.device), q], dim=1)
        g = (vq.T @ vq).cpu().numpy()
    else:
        vq = np.hstack([np.asarray(v), np.asarray(q)])
        g = vq.conj().T @ vq
    return float(np.max(np.abs(np.linalg.eigvalsh(g) - 1.0))) if g.size else 0.0
