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


def _defect_then(v, exc, orth_tol=1e-8):
    """The reference validates the orthonormality of v (reflector.py:220-223)
    before the seed's choice / p checks (reflector.py:178-204) and before the
    intra dispatch (twostage.py:54): raise OrthonormalityError if the device
    defect exceeds orth_tol, else the deferred error `exc`."""
    from .core import orthonormality_defect
    defect = orthonormality_defect(v)
    if defect > orth_tol:
        raise E.OrthonormalityError(f"||v^* v - I||_2 = {defect:.3e} exceeds {orth_tol:.1e}")
    raise exc


def _run_two_stage(dev, V, A, Q, R, S, choice, intra, P, cplx, gram=None):
    """One C-ABI call on device matrices (DMat); returns the diagnostics.
    gram: optional device tensor holding V^T V (real only)."""
    ctx = D.ctx(dev)
    diag = (C.c_double * 3)()
    if gram is not None:
        rc = lib().ots_two_stage_gram_f64(
            ctx, A.rows, V.cols, A.cols, V.ptr, V.ld, A.ptr, A.ld, CHOICES[choice],
            INTRA[intra], P.ptr if P is not None else None, P.ld if P is not None else 0,
            1e-8, 0, C.c_void_p(gram.data_ptr()), gram.stride(0), Q.ptr, Q.ld, R.ptr, R.ld, S.ptr, S.ld, diag,
            D.stream_ptr(dev))
        check(rc, ctx)
        return ReflectorDiagnostics(float(diag[0]), float(diag[1]))
    fn = lib().ots_two_stage_c128 if cplx else lib().ots_two_stage_f64
    rc = fn(
        ctx, A.rows, V.cols, A.cols, V.ptr, V.ld, A.ptr, A.ld, CHOICES[choice],
        INTRA[intra], P.ptr if P is not None else None, P.ld if P is not None else 0,
        1e-8, 0, Q.ptr, Q.ld, R.ptr, R.ld, S.ptr, S.ld, diag, D.stream_ptr(dev))
    check(rc, ctx)   # OrthonormalityError before the non-finite ValueError (device-side order)
    return ReflectorDiagnostics(float(diag[0]), float(diag[1]))


def two_stage_qr(v, a, choice="qr", intra="householder", p=None):
    """Orthogonalize a against orthonormal v in two stages (Algorithm 1).

    Returns TwoStageResult(q, r, s, diagnostics) with
    [v, a] = [v, q] [[I, s], [0, r]] and [v, q]^* [v, q] = I.
    numpy in -> numpy out; CUDA tensors in -> CUDA tensors out (zero-copy).
    Validation order of the reference: DimensionError (twostage.py:77-80),
    OrthonormalityError (reflector.py:220-223), seed / choice / p errors
    (reflector.py:178-204), non-finite ValueError (core.py:72-73), unknown
    intra (twostage.py:54).
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
        _defect_then(v, E.ParameterError(f"unknown choice {choice!r}; expected one of "
                                         f"('mlu', 'qr', 'polar', 'explicit')"))
    if choice == "explicit":
        if p is None:
            _defect_then(v, E.ParameterError("choice='explicit' requires a seed matrix p"))
        try:
            p = as_matrix(p, "p")
        except E.DimensionError as exc:
            _defect_then(v, exc)
        if tuple(p.shape) != (k0, k0):
            _defect_then(v, E.DimensionError(f"seed p must be {k0}x{k0}, got {tuple(p.shape)}"))
    if intra not in INTRA:
        bad = E.ParameterError(f"unknown intra method {intra!r}; expected {INTRA_METHODS}")
        try:   # every earlier error of the reference's order, then the intra dispatch
            two_stage_qr(v, a, choice, "householder", p)
        except ValueError:
            raise bad from None
        raise bad
    if k > 64:
        return _two_stage_wide(v, a, choice, intra, p, was_torch)
    dev = D.pick_device(v, a)
    todev = D.cto_device if cplx else D.to_device
    V = todev(v, dev)
    A = todev(a, dev)
    P = todev(p, dev) if choice == "explicit" else None
    if cplx:
        Q, R, S = D.cempty(n, k, dev), D.czeros(k, k, dev), D.cempty(k0, k, dev)
    else:
        Q, R, S = D.empty(n, k, dev), D.zeros(k, k, dev), D.empty(k0, k, dev)
    diag = _run_two_stage(dev, V, A, Q, R, S, choice, intra, P, cplx)
    return TwoStageResult(Q.view() if was_torch else Q.numpy(),
                          R.view() if was_torch else R.numpy(),
                          S.view() if was_torch else S.numpy(), diag)


def _two_stage_wide(v, a, choice, intra, p, was_torch):
    """k > 64: the reference's own sequence (twostage.py:90-97) on device
    primitives -- reflector object (seed, T, W_t), H^* A through the DMMA
    streaming kernels, S = P^* (H^* A)_top, the column-blocked intra QR with
    LAPACK signs (core._householder_qr_wide), Q = H [0; Q_], diagnostics
    from k0 x k0 data."""
    from .core import gram
    from .reflector import apply_reflector, build_reflector, reflector_diagnostics
    t = D.torch()
    n, k0 = v.shape
    k = a.shape[1]
    dt = t.complex128 if (is_complex(v) or is_complex(a)) else t.float64
    dev = D.pick_device(v, a)
    vd = (v if D.is_torch(v) else t.from_numpy(v)).to(device=f"cuda:{dev}", dtype=dt).contiguous()
    ad = (a if D.is_torch(a) else t.from_numpy(a)).to(device=f"cuda:{dev}", dtype=dt)
    h = build_reflector(vd, choice, p)
    ah = apply_reflector(h, ad, adjoint=True)
    pm = (h.p if D.is_torch(h.p) else t.from_numpy(np.ascontiguousarray(h.p))).to(device=f"cuda:{dev}", dtype=dt)
    s = gram(pm, ah[:k0])                                   # P^* (H^* A)_top  (twostage.py:92)
    qr = intra_qr(ah[k0:].contiguous(), intra)
    lifted = t.zeros((n, k), dtype=dt, device=f"cuda:{dev}")
    lifted[k0:] = qr.q
    q = apply_reflector(h, lifted)
    diag = reflector_diagnostics(h)
    r = qr.r
    if was_torch:
        return TwoStageResult(q, r, s, diag)
    return TwoStageResult(q.cpu().numpy(), r.cpu().numpy() if D.is_torch(r) else r, s.cpu().numpy(), diag)


class KrylovBasis:
    """Device-resident growing orthonormal basis [Q_0 ... Q_i] -- the state of
    the Alg. 3 / block-Krylov driver (twostage.py:100-151, BASELINE configs[4]).
    One preallocated n x capacity buffer: `append(a)` orthogonalises the
    block a against the current basis with Algorithm 1, reading V as a
    column view of the buffer and writing Q straight into the next columns
    (no per-block concatenation, ref :132); it returns the block's (q, r, s,
    diagnostics).  incremental_gram (real data): the Gram of the basis is
    kept on the device and extended per block by [Q_acc, Q_i]^T Q_i (one pass
    with k_i output columns) instead of the full V^T V in every call; the
    orthonormality check, seed and diagnostics read it (V does not change
    between blocks, so the values agree up to rounding)."""

    def __init__(self, n, capacity, dtype="float64", device=None, choice="qr", intra="householder",
                 incremental_gram=False):
        t = D.torch()
        self.cplx = str(dtype).endswith("complex128")
        self.dt = t.complex128 if self.cplx else t.float64
        self.dev = D.pick_device() if device is None else int(device)
        self.n, self.cap, self.m = n, capacity, 0
        self.choice, self.intra = choice, intra
        self.ldb = max(2, capacity + (capacity & 1))
        self.buf = t.empty((max(n, 1), self.ldb), dtype=self.dt, device=f"cuda:{self.dev}")
        self.inc = incremental_gram and not self.cplx
        self.G = t.zeros((capacity, capacity + (capacity & 1)), dtype=t.float64,
                         device=f"cuda:{self.dev}") if self.inc else None

    @property
    def q(self):
        return self.buf[:, :self.m] if self.n else self.buf[:0, :self.m]

    def _grow_gram(self, m, ki):
        from .core import gram as _gram
        if not self.inc:
            return
        if m == 0:
            self.G[:ki, :ki] = _gram(self.buf[:, :ki])
            return
        cross = _gram(self.buf[:, :m + ki], self.buf[:, m:m + ki])       # [Q_acc, Q_i]^T Q_i
        self.G[:m + ki, m:m + ki] = cross
        self.G[m:m + ki, :m] = cross[:m].T

    def append(self, a):
        t = D.torch()
        a = a if D.is_torch(a) else t.from_numpy(np.ascontiguousarray(a))
        a = a.to(device=f"cuda:{self.dev}", dtype=self.dt)
        ki, m = a.shape[1], self.m
        if a.shape[0] != self.n:
            raise E.DimensionError("all blocks must have the same row count")
        if m + ki > self.cap:
            raise E.DimensionError(f"basis capacity {self.cap} exceeded")
        if m == 0:
            qr = intra_qr(a, self.intra)
            self.buf[:, :ki] = qr.q
            self.m = ki
            self._grow_gram(0, ki)
            z = t.zeros((0, ki), dtype=self.dt, device=a.device)
            return TwoStageResult(self.buf[:, :ki], qr.r, z, ReflectorDiagnostics(1.0, 0.0))
        if ki == 0:
            z = t.zeros((0, 0), dtype=self.dt, device=a.device)
            return TwoStageResult(self.buf[:, m:m], z, t.zeros((m, 0), dtype=self.dt, device=a.device),
                                  ReflectorDiagnostics(1.0, 0.0))
        todev = D.cto_device if self.cplx else D.to_device
        V = D.DMat(self.buf, m, ld=self.ldb)         # column view [Q_0 ... Q_{i-1}]
        A = todev(a, self.dev)
        direct = (m % 2 == 0) or self.cplx           # Q view 16-byte aligned
        if direct:
            Q = D.DMat(self.buf[:, m:], ki, ld=self.ldb)
        else:
            Q = (D.cempty if self.cplx else D.empty)(self.n, ki, self.dev)
        if self.cplx:
            R, S = D.czeros(ki, ki, self.dev), D.cempty(m, ki, self.dev)
        else:
            R, S = D.zeros(ki, ki, self.dev), D.empty(m, ki, self.dev)
        diag = _run_two_stage(self.dev, V, A, Q, R, S, self.choice, self.intra, None, self.cplx,
                              gram=self.G[:m, :m] if self.inc else None)
        if not direct:
            self.buf[:, m:m + ki] = Q.view()
        self.m = m + ki
        self._grow_gram(m, ki)
        return TwoStageResult(self.buf[:, m:m + ki], R.view(), S.view(), diag)


def block_householder_qr(blocks, choice="qr", intra="householder", incremental_gram=False):
    """Algorithm 3 driver (twostage.py:100-151): block 0 by the intra QR,
    block i >= 1 by Algorithm 1 against the accumulated Q, on a
    device-resident `KrylovBasis` (see there; incremental_gram is its
    extension).  numpy blocks are moved to the device once and the results
    copied back at the end."""
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
    cplx = any(is_complex(b) for b in blocks)       # ref :117 np.result_type(*blocks)
    t = D.torch()
    dev = D.pick_device(*blocks)
    kb = KrylovBasis(n, total, "complex128" if cplx else "float64", dev, choice, intra, incremental_gram)
    r_full = t.zeros((total, total), dtype=kb.dt, device=f"cuda:{dev}")
    worst = ReflectorDiagnostics(1.0, 0.0)
    offset = 0
    for i, blk in enumerate(blocks):
        ki = sizes[i]
        try:
            res = kb.append(blk)
        except E.IntraFailure as exc:
            exc.block = i
            raise
        if offset:
            r_full[:offset, offset:offset + ki] = res.s
        r_full[offset:offset + ki, offset:offset + ki] = res.r
        if i and res.diagnostics.kappa_t > worst.kappa_t:
            worst = res.diagnostics
        offset += ki
    q = kb.q
    if was_torch:
        return BlockQRResult(q, r_full, sizes, worst)
    return BlockQRResult(q.cpu().numpy(), r_full.cpu().numpy(), sizes, worst)


def reorthogonalized_two_stage(v, a, choice="qr", intra="householder", sweeps=1, sequence=None):
    """twostage.py:154-180: repeated Algorithm-1 passes composing r and s,
    or (choice="bcgs") the classical inter/intra step sequence of the
    baselines (baselines.py:34-73) on the GPU."""
    if choice == "bcgs":
        from .baselines import bcgs_two_stage
        return bcgs_two_stage(v, a, sequence or ["inter", "intra"], intra=intra)
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
    """orthonormality_defect([v, q]) (twostage.py:183-184) on the GPU: the
    Gram of the stacked block and its symmetric spectrum (complex-aware)."""
    from .core import orthonormality_defect
    if D.is_torch(v) or D.is_torch(q):
        t = D.torch()
        dev = q.device if D.is_torch(q) else v.device
        vq = t.cat([t.as_tensor(v, device=dev), t.as_tensor(q, device=dev)], dim=1)
    else:
        vq = np.hstack([np.asarray(v), np.asarray(q)])
    return orthonormality_defect(vq)
