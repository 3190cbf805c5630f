"""Classical comparators of the two-stage method on the GPU (baselines.py of
the reference): BCGS inter/intra step sequences, BCGS2, BMGS (plain and WY)
and the two-stage Cholesky-QR.  SURVEY 8(f) rank 4: the fast-but-unstable
comparators for the Fig.-2 timing analogue (`timing_mode`).

Every n-length product runs on the DMMA streaming kernels of the path
(`ots_gram_*` for c = v^* x, `ots_update_*` for x - v c; the intra QR is the
device TSQR / shifted Cholesky-QR).  The only other arithmetic is on k x k /
k0 x k blocks (Cholesky of the CholQR Gram, products composing R and S),
which stays on the device as small torch ops.  numpy in -> numpy out, CUDA
tensors in -> CUDA tensors out."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import errors as E
from .core import as_matrix, gram, householder_qr, is_complex, orthonormality_defect, update
from .twostage import BlockQRResult, TwoStageResult, intra_qr

SCHEMES = ("BCGS", "BCGS2", "BMGS", "BMGS_WY", "CholQR2Stage")


@dataclass
class BaselineSpec:
    """baselines.py:20-32."""
    scheme: str = "BCGS"
    intra: str = "householder"
    reorth_sequence: list = field(default_factory=lambda: ["inter", "intra"])

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise E.ParameterError(f"unknown scheme {self.scheme!r}")
        if not self.reorth_sequence:
            raise E.ParameterError("reorth_sequence must be nonempty")
        if self.reorth_sequence[-1] != "intra":
            raise E.ParameterError("reorth_sequence must end with an intra step")


def _prep(*xs):
    """device tensors of a common dtype; returns (tensors, was_torch, dev, cplx)."""
    t = D.torch()
    was_torch = any(D.is_torch(x) for x in xs if x is not None)
    cplx = any(is_complex(x) for x in xs if x is not None)
    dev = D.pick_device(*[x for x in xs if x is not None])
    dt = t.complex128 if cplx else t.float64
    out = []
    for x in xs:
        if x is None:
            out.append(None)
            continue
        x = as_matrix(x, "x")
        x = x if D.is_torch(x) else t.from_numpy(x)
        out.append(x.to(device=f"cuda:{dev}", dtype=dt))
    return out, was_torch, dev, cplx


def _out(x, was_torch):
    return x if was_torch else x.cpu().numpy()


def _hstack(xs):
    return D.torch().cat(xs, dim=1)


def bcgs_two_stage(v, a, spec=None, intra=None):
    """baselines.py:34-73: run an inter/intra step sequence of the classical
    block scheme, maintaining a = v s + work r; sweep_history holds the
    augmented defect after each intra step."""
    if D.is_torch(v) or D.is_torch(a):
        if v.dim() != 2 or a.dim() != 2:
            raise E.DimensionError("v and a must be 2-D")
    else:
        v, a = as_matrix(v, "v"), as_matrix(a, "a")
    if v.shape[0] != a.shape[0]:
        raise E.DimensionError("v and a must have the same row count")
    if isinstance(spec, BaselineSpec):
        sequence = spec.reorth_sequence
        intra = intra or spec.intra
    else:
        sequence = spec or ["inter", "intra"]
    intra = intra or "householder"
    if not sequence or sequence[-1] != "intra":
        raise E.ParameterError("sequence must be nonempty and end with 'intra'")
    (v, a), was_torch, dev, cplx = _prep(v, a)
    t = D.torch()
    k0, k = v.shape[1], a.shape[1]
    work = a
    s = t.zeros((k0, k), dtype=a.dtype, device=a.device)
    r = t.eye(k, dtype=a.dtype, device=a.device)
    history = []
    for step in sequence:
        if step == "inter":
            c = gram(v, work)                       # v^* work
            work = update(v, -c, work)              # work - v c
            s = s + c @ r
        elif step == "intra":
            qr = intra_qr(work, intra)
            work = qr.q
            r = qr.r @ r
            history.append(orthonormality_defect(_hstack([v, work])))
        else:
            raise E.ParameterError(f"unknown step {step!r}")
    return TwoStageResult(_out(work, was_torch), _out(r, was_torch), _out(s, was_torch), None,
                          sweep_history=history)


def _b_apply(inner, x):
    return x if inner is None or inner.kind == "euclidean" else inner.apply(x)


def b_intra_qr(x, inner, intra="householder"):
    """oblique.py:241-276 (the baselines' intra step under a B inner product):
    householder = Euclidean QR, then a Cholesky correction of the B-Gram;
    cholshift = shifted Cholesky-QR on the B-Gram plus two unshifted passes.
    Breakdown raises IntraFailure."""
    from .oblique import _tcholesky
    t = D.torch()
    (x,), was_torch, dev, cplx = _prep(x)
    m, n = x.shape
    try:
        if intra == "householder":
            qe = householder_qr(x)
            g = gram(qe.q, _b_apply(inner, qe.q))
            l = _tcholesky(g)
            linv = t.linalg.solve_triangular(l, t.eye(n, dtype=l.dtype, device=l.device), upper=False)
            q = update(qe.q, linv.mH)
            return _qrpair(q, t.triu(l.mH @ qe.r), was_torch)
        if intra == "cholshift":
            if n == 0:
                return _qrpair(x.clone(), t.zeros((0, 0), dtype=x.dtype, device=x.device), was_torch)
            from .core import EPS
            g = gram(x, _b_apply(inner, x))
            g = (g + g.mH) / 2.0
            from .core import spectral_norm
            shift = 11.0 * (m * n + n * (n + 1)) * EPS * spectral_norm(g)
            l = _tcholesky(g + shift * t.eye(n, dtype=g.dtype, device=g.device))
            q = update(x, _inv_h(l))
            r = l.mH
            for _ in range(2):
                g2 = gram(q, _b_apply(inner, q))
                g2 = (g2 + g2.mH) / 2.0
                l2 = _tcholesky(g2)
                q = update(q, _inv_h(l2))
                r = l2.mH @ r
            return _qrpair(q, t.triu(r), was_torch)
    except E.NotPositiveDefinite as exc:
        raise E.IntraFailure(f"intra B-orthogonalization broke down: {exc}") from None
    raise E.ParameterError(f"unknown intra method {intra!r}")


def _inv_h(l):
    """L^{-H} for lower-triangular L (k x k, device)."""
    t = D.torch()
    n = l.shape[0]
    return t.linalg.solve_triangular(l, t.eye(n, dtype=l.dtype, device=l.device), upper=False).mH


def _qrpair(q, r, was_torch):
    from .core import QRPair
    return QRPair(_out(q, was_torch), _out(r, was_torch))


def bcgs2_block(blocks, intra="householder", inner=None):
    """baselines.py:76-125: two-sweep (inter, intra, inter, intra) block CGS;
    with a weighted inner product the projections and the intra step run
    under it.  Intra breakdown raises IntraFailure tagged with the block."""
    if not blocks:
        raise E.ParameterError("need at least one block")
    blocks, was_torch, dev, cplx = _prep(*blocks)
    n = blocks[0].shape[0]
    sizes = [b.shape[1] for b in blocks]
    total = sum(sizes)
    if total > n:
        raise E.DimensionError(f"need sum(k_i) <= n, got {total} > {n}")
    euclid = inner is None or inner.kind == "euclidean"
    t = D.torch()

    def _intra(x, idx):
        try:
            if euclid:
                return intra_qr(x, intra)
            return b_intra_qr(x, inner, intra)
        except E.IntraFailure as exc:
            exc.block = idx
            raise

    r_full = t.zeros((total, total), dtype=blocks[0].dtype, device=blocks[0].device)
    qr0 = _intra(blocks[0], 0)
    qs = [_tq(qr0.q, dev)]
    r_full[:sizes[0], :sizes[0]] = _tq(qr0.r, dev)
    offset = sizes[0]
    for i in range(1, len(blocks)):
        ki = sizes[i]
        qacc = _hstack(qs)
        s1 = gram(qacc, _b_apply(inner, blocks[i]))
        y = update(qacc, -s1, blocks[i])
        qr1 = _intra(y, i)
        q1, r1 = _tq(qr1.q, dev), _tq(qr1.r, dev)
        s2 = gram(qacc, _b_apply(inner, q1))
        z = update(qacc, -s2, q1)
        qr2 = _intra(z, i)
        qs.append(_tq(qr2.q, dev))
        m = offset
        r_full[:m, offset:offset + ki] = s1 + s2 @ r1
        r_full[offset:offset + ki, offset:offset + ki] = _tq(qr2.r, dev) @ r1
        offset += ki
    return BlockQRResult(_out(_hstack(qs), was_torch), _out(r_full, was_torch), sizes)


def _tq(x, dev):
    t = D.torch()
    return x if D.is_torch(x) else t.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{dev}")


def bmgs_inter(v_blocks, a, wy=False):
    """baselines.py:128-156: block-MGS projection of a against [v_1 ... v_p];
    WY mode assembles the lower-triangular correction T and applies
    I - V T V^* in two products."""
    if not v_blocks:
        raise E.ParameterError("need at least one v block")
    (a, *v_blocks), was_torch, dev, cplx = _prep(a, *v_blocks)
    n = a.shape[0]
    if any(b.shape[0] != n for b in v_blocks):
        raise E.DimensionError("v blocks and a must share the row count")
    t = D.torch()
    if not wy:
        work = a.clone()
        for vb in v_blocks:
            work = update(vb, -gram(vb, work), work)
        return _out(work, was_torch)
    vcat = _hstack(v_blocks)
    m = vcat.shape[1]
    tm = t.eye(m, dtype=a.dtype, device=a.device)
    offset = v_blocks[0].shape[1]
    for i in range(1, len(v_blocks)):
        ki = v_blocks[i].shape[1]
        tm[offset:offset + ki, :offset] = -gram(v_blocks[i], vcat[:, :offset]) @ tm[:offset, :offset]
        offset += ki
    return _out(update(vcat, -(tm @ gram(vcat, a)), a), was_torch)


def cholqr_two_stage(v, a):
    """baselines.py:159-175: Cholesky-QR of [v, a] exploiting v's
    orthonormality: r^* = chol(a^* a - (a^* v)(v^* a)); NotPositiveDefinite
    when that Gram complement is numerically indefinite."""
    from .oblique import _tcholesky
    (v, a), was_torch, dev, cplx = _prep(v, a)
    if v.shape[0] != a.shape[0]:
        raise E.DimensionError("v and a must have the same row count")
    t = D.torch()
    s = gram(v, a)
    g = gram(a) - s.mH @ s
    g = (g + g.mH) / 2.0
    l = _tcholesky(g)
    q = update(update(v, -s, a), _inv_h(l))
    return TwoStageResult(_out(q, was_torch), _out(t.triu(l.mH), was_torch), _out(s, was_torch), None)


def timing_mode(config=None, out=None):
    """Fig.-2 timing analogue (experiments.py:280-318): median-of-`reps` times
    per scheme relative to one Householder QR of the stacked [v, a], here on
    the GPU with device-resident inputs (CUDA events around each call, the
    result's copy back excluded).  Rows carry the reference's keys; the
    comparators BCGS2 (two inter/intra sweeps) and CholQR2Stage are added.
    `out` (optional): CSV path."""
    from . import workloads as W
    from .core import householder_qr as hqr
    from .twostage import two_stage_qr
    t = D.torch()
    config = dict(config or {})
    n = config.get("n", 10000)
    k0 = config.get("k0", 100)
    k = config.get("k", 100)
    reps = config.get("reps", 5)
    choices = config.get("choices", ["mlu", "qr", "polar"])
    seed = config.get("seed", 1)
    fld = config.get("field", "real")
    dev = t.cuda.current_device()
    v = hqr(t.from_numpy(W.normal_matrix(W.make_rng(seed), n, k0, fld)).to(f"cuda:{dev}")).q
    a = t.from_numpy(W.normal_matrix(W.make_rng(seed + 40009), n, k, fld)).to(f"cuda:{dev}")
    stacked = t.cat([v, a], dim=1).contiguous()

    def _median_ms(fn):
        fn()
        times = []
        for _ in range(reps):
            e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            t.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return float(np.median(times))

    naive = _median_ms(lambda: hqr(stacked))
    rows = [{"scheme": "householder_full", "choice": "", "intra": "householder", "n": n, "k0": k0, "k": k,
             "wall_ms": naive, "rel_time": 1.0}]
    for choice in choices:
        ms = _median_ms(lambda: two_stage_qr(v, a, choice))
        rows.append({"scheme": "twostage", "choice": choice, "intra": "householder", "n": n, "k0": k0, "k": k,
                     "wall_ms": ms, "rel_time": ms / naive})
    for scheme, fn in (("BCGS2", lambda: bcgs_two_stage(v, a, ["inter", "intra", "inter", "intra"])),
                       ("CholQR2Stage", lambda: cholqr_two_stage(v, a))):
        try:
            ms = _median_ms(fn)
        except (E.NotPositiveDefinite, E.IntraFailure):
            ms = float("nan")
        rows.append({"scheme": scheme, "choice": "", "intra": "householder", "n": n, "k0": k0, "k": k,
                     "wall_ms": ms, "rel_time": ms / naive})
    if out:
        import csv
        cols = ["scheme", "choice", "intra", "n", "k0", "k", "wall_ms", "rel_time"]
        with open(out, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=cols)
            w.writeheader()
            for row in rows:
                w.writerow(row)
    return rows
