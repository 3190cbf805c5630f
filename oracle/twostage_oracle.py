"""CPU ORACLE for the two-stage Householder orthogonalization hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2602_14449_b200/`) imports, links or executes this file.  It is used
as the *checker* by `tests/`, by `__graft_entry__.smoke()`, and by
`bench.py`'s `cpu_baseline` leg / `--impl reference` arm (the reference's
own CPU algorithm timed on the host cores).

What it is: a numpy/scipy restatement of the reference package
`orthoqr` 0.1.0 (`/root/reference/pkg/src/orthoqr`, pure Python) for the
path named by BASELINE.json's north_star:

  * Algorithm 1 `two_stage_qr`            -- twostage.py:57-97
  * seeds mlu / qr / polar / explicit      -- reflector.py:174-204
  * the pivot-free modified LU (Alg. 2)    -- reflector.py:53-77
  * T-solvers                              -- reflector.py:80-153
  * reflector build / apply / diagnostics  -- reflector.py:207-247
  * intra QR (householder / cholshift)     -- twostage.py:45-54, core.py:61-84,177-202
  * B-inner Algorithm 4 `b_two_stage_qr`   -- oblique.py:93-315
  * Algorithm 3 driver                     -- twostage.py:100-151
  * metrics                                -- metrics.py:25-73

The dense arithmetic underneath lives in third-party LAPACK, exactly as in
the reference: numpy 2.3.5 `linalg.qr` (dgeqrf/zgeqrf + dorgqr/zungqr),
`linalg.svd` (gesdd) and scipy 1.18.1 `solve_triangular` (trtrs),
`cholesky` (potrf), `lu_factor/lu_solve` (getrf/getrs), all on OpenBLAS
0.3.30 / 0.3.31.dev.  Those published LAPACK algorithms are called, not
re-derived (they are present on the GPU box as well).

Pinning: `tests/golden/make_golden.py` ran the real reference in the build
container and stored its outputs as `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this restatement against every fixture
(and the SPEC.md known-answer examples) before any GPU parity test trusts it.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla

U_ROUND = 2.0 ** -53  # core.py:22


class OracleError(Exception):
    """Raised with the reference's exception *class name* in `.kind`."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


# ----------------------------------------------------------------------------
# dense helpers (core.py)
# ----------------------------------------------------------------------------

def to_dense(x, name="matrix"):
    """core.py:25-32: 2-D check, contiguous float64 or complex128."""
    x = np.asarray(x)
    if x.ndim != 2:
        raise OracleError("DimensionError", f"{name} must be 2-D, got shape {x.shape}")
    dt = np.complex128 if np.iscomplexobj(x) else np.float64
    return np.ascontiguousarray(x, dtype=dt)


def norm2(x):
    """core.py:35-40: largest singular value (0 for empty)."""
    x = np.asarray(x)
    return 0.0 if x.size == 0 else float(np.linalg.norm(x, 2))


def gram_defect(x):
    """core.py:43-49: ||x^* x - I||_2."""
    x = np.asarray(x)
    if x.size == 0:
        return 0.0
    g = x.conj().T @ x
    g[np.diag_indices_from(g)] -= 1.0
    return norm2(g)


def lapack_qr(x, nonneg=False):
    """core.py:61-84.  LAPACK geqrf/orgqr; optional phase fix making diag(R)
    real and >= 0 (a zero diagonal keeps phase 1).  Returns (Q, triu(R))."""
    x = to_dense(x, "a")
    m, c = x.shape
    if m < c:
        raise OracleError("DimensionError", f"need rows >= cols, got {m}x{c}")
    if x.size and not np.isfinite(x).all():
        raise ValueError("input contains non-finite entries")
    q, r = np.linalg.qr(x, mode="reduced")
    if nonneg and c:
        d = np.diag(r).copy()
        mag = np.abs(d)
        ph = np.ones_like(d)
        nz = mag != 0
        ph[nz] = d[nz] / mag[nz]
        q = q * ph[None, :]
        r = r / ph[:, None]
        r[np.arange(c), np.arange(c)] = mag
    return q, np.triu(r)


def herm_chol(x):
    """core.py:87-105: Hermitian check at 1e-12*||x||, symmetrize, potrf."""
    x = to_dense(x, "a")
    if x.shape[0] != x.shape[1]:
        raise OracleError("DimensionError", f"cholesky needs a square matrix, got {x.shape}")
    if x.shape[0] == 0:
        return x.copy()
    if norm2(x - x.conj().T) > 1e-12 * norm2(x):
        raise OracleError("NotHermitian", "matrix is not Hermitian to 1e-12 * ||a||_2")
    try:
        return sla.cholesky(0.5 * (x + x.conj().T), lower=True, check_finite=True)
    except sla.LinAlgError as exc:
        raise OracleError("NotPositiveDefinite", str(exc)) from None


def polar_split(x):
    """core.py:108-120: SVD polar, U = u vh, H = V S V^* symmetrized."""
    x = to_dense(x, "a")
    u, s, vh = np.linalg.svd(x)
    h = (vh.conj().T * s) @ vh
    return u @ vh, 0.5 * (h + h.conj().T)


def cond_2(x):
    """core.py:123-134."""
    s = np.linalg.svd(to_dense(x, "a"), compute_uv=False)
    return float("inf") if s[-1] == 0.0 else float(s[0] / s[-1])


def trsolve(t, b, lower, adjoint=False, unit=False):
    """core.py:137-156 (left side only -- all the path needs)."""
    if not unit and t.shape[0] and (np.diag(t) == 0).any():
        raise OracleError("SingularError", "zero diagonal entry in triangular factor")
    return sla.solve_triangular(t, b, lower=lower, trans="C" if adjoint else "N",
                                unit_diagonal=unit, check_finite=False)


def cholqr_shifted(x, passes=2):
    """core.py:177-202: shifted CholeskyQR + `passes` unshifted refinements."""
    x = to_dense(x, "a")
    m, c = x.shape
    if m < c:
        raise OracleError("DimensionError", f"need rows >= cols, got {m}x{c}")
    if c == 0:
        return x.copy(), np.zeros((0, 0), dtype=x.dtype)
    g = x.conj().T @ x
    g = 0.5 * (g + g.conj().T)
    g = g + 11.0 * (m * c + c * (c + 1)) * U_ROUND * norm2(g) * np.eye(c)
    lo = herm_chol(g)
    q = trsolve(lo, x.conj().T, lower=True).conj().T
    r = lo.conj().T
    for _ in range(passes):
        g2 = q.conj().T @ q
        lo = herm_chol(0.5 * (g2 + g2.conj().T))
        q = trsolve(lo, q.conj().T, lower=True).conj().T
        r = lo.conj().T @ r
    return q, np.triu(r)


# ----------------------------------------------------------------------------
# Algorithm 2 and the seed / T constructions (reflector.py)
# ----------------------------------------------------------------------------

def mlu(z):
    """reflector.py:53-77 (paper Alg. 2).

    Pivot-free LU of diag(p) - z with p_i = -sign(z_ii), sign(mu)=+1 iff
    Re mu >= 0.  Returns (p, L unit-lower, U upper)."""
    z = to_dense(z, "z")
    n = z.shape[0]
    if z.shape[0] != z.shape[1]:
        raise OracleError("DimensionError", f"modified_lu needs a square matrix, got {z.shape}")
    if norm2(z) > 1.0 + 1e-8:
        raise OracleError("NormBoundError", "||z||_2 exceeds 1 beyond tolerance")
    s = z.copy()
    p = np.empty(n)
    lo = np.eye(n, dtype=z.dtype)
    up = np.zeros((n, n), dtype=z.dtype)
    for j in range(n):
        p[j] = 1.0 if s[j, j].real < 0 else -1.0
        up[j, j] = p[j] - s[j, j]
        up[j, j + 1:] = -s[j, j + 1:]
        lo[j + 1:, j] = -s[j + 1:, j] / up[j, j]
        s[j + 1:, j + 1:] += lo[j + 1:, j, None] * up[None, j, j + 1:]
    return p, lo, up


class TFactor:
    """T of the reflector with its natural solver (reflector.py:80-153).

    kind: "mlu" (T = (LU)^* diag(p)), "tri" (lower-triangular T),
    "chol" (HPD T via Cholesky), "lu" (dense T, pivoted LU)."""

    def __init__(self, kind, **kw):
        self.kind = kind
        self.__dict__.update(kw)
        if kind == "chol":
            self.lo = herm_chol(self.t)
        elif kind == "lu":
            self.lu, self.piv = sla.lu_factor(self.t, check_finite=False)
            if (np.diag(self.lu) == 0).any():
                raise OracleError("SingularTError", "T is numerically singular")

    def dense(self):
        if self.kind == "mlu":
            return (self.lo @ self.up).conj().T * self.p[None, :]
        return self.t

    def solve(self, b, adjoint=False):
        """T^{-1} b, or T^{-*} b."""
        b = np.asarray(b)
        if self.kind == "mlu":                       # reflector.py:88-98
            if adjoint:
                y = trsolve(self.lo, self.p[:, None] * b, lower=True, unit=True)
                return trsolve(self.up, y, lower=False)
            y = trsolve(self.up, b, lower=False, adjoint=True)
            y = trsolve(self.lo, y, lower=True, adjoint=True, unit=True)
            return self.p[:, None] * y
        if self.kind == "tri":                       # reflector.py:112-113
            return trsolve(self.t, b, lower=True, adjoint=adjoint)
        if self.kind == "chol":                      # reflector.py:128-131
            return trsolve(self.lo, trsolve(self.lo, b, lower=True), lower=True, adjoint=True)
        return sla.lu_solve((self.lu, self.piv), b, trans=2 if adjoint else 0,
                            check_finite=False)      # reflector.py:148-150


def seed(z, choice, p=None):
    """reflector.py:174-204: (P, TFactor) for T = I - z^* P."""
    n = z.shape[0]
    eye = np.eye(n, dtype=z.dtype)
    if choice == "mlu":
        pd, lo, up = mlu(z)
        return np.diag(pd).astype(z.dtype), TFactor("mlu", p=pd, lo=lo, up=up)
    if choice == "qr":
        q1, r1 = lapack_qr(z, nonneg=True)
        return -q1, TFactor("tri", t=eye + r1.conj().T)
    if choice == "polar":
        u, h = polar_split(z)
        return -u, TFactor("chol", t=eye + h)
    if choice == "explicit":
        if p is None:
            raise OracleError("ParameterError", "choice='explicit' requires a seed matrix p")
        p = to_dense(p, "p")
        if p.shape != (n, n):
            raise OracleError("DimensionError", f"seed p must be {n}x{n}, got {p.shape}")
        if gram_defect(p) > 1e-12 * max(n, 1):
            raise OracleError("ParameterError", "explicit seed p is not unitary to tolerance")
        t = np.eye(n, dtype=np.result_type(z, p)) - z.conj().T @ p
        return p, TFactor("lu", t=t)
    raise OracleError("ParameterError", f"unknown choice {choice!r}")


class Reflector:
    """H = I - W T^{-1} W^*, W = [P;0] - V (reflector.py:156-165,207-228)."""

    def __init__(self, v, choice="qr", p=None, orth_tol=1e-8, allow_defect=False):
        v = to_dense(v, "v")
        n, k0 = v.shape
        if k0 > n:
            raise OracleError("DimensionError", f"v must be tall, got {v.shape}")
        if k0 == 0:
            raise OracleError("DimensionError", "v must have at least one column")
        self.defect = gram_defect(v)
        if self.defect > orth_tol and not allow_defect:
            raise OracleError("OrthonormalityError",
                              f"||v^* v - I||_2 = {self.defect:.3e} exceeds {orth_tol:.1e}")
        self.p, self.tf = seed(v[:k0], choice, p)
        self.w = -v
        self.w[:k0] += self.p            # W_top = fl(P - V_top), rounded once
        self.n, self.k0, self.choice = n, k0, choice

    def apply(self, x, adjoint=False):
        """reflector.py:231-238: x - W T^{-(*)} (W^* x)."""
        x = to_dense(x, "x")
        if x.shape[0] != self.n:
            raise OracleError("DimensionError", "row mismatch")
        return x - self.w @ self.tf.solve(self.w.conj().T @ x, adjoint=adjoint)

    def diagnostics(self):
        """reflector.py:241-247: kappa_2(T) and ||W T^{-1}||_2 (k0 x n solve)."""
        kt = cond_2(self.tf.dense())
        z = self.tf.solve(self.w.conj().T, adjoint=True)
        return kt, norm2(z)


# ----------------------------------------------------------------------------
# Algorithm 1 (twostage.py)
# ----------------------------------------------------------------------------

def intra(x, method="householder"):
    """twostage.py:45-54."""
    if method == "householder":
        return lapack_qr(x)
    if method == "cholshift":
        try:
            return cholqr_shifted(x)
        except OracleError as exc:
            if exc.kind == "NotPositiveDefinite":
                raise OracleError("IntraFailure", f"shifted Cholesky-QR broke down: {exc}") from None
            raise
    raise OracleError("ParameterError", f"unknown intra method {method!r}")


def two_stage(v, a, choice="qr", intra_method="householder", p=None, diagnostics=True):
    """twostage.py:57-97 (paper Alg. 1).

    Returns dict(q, r, s, kappa_t, wt_inv_norm, defect)."""
    v = to_dense(v, "v")
    a = to_dense(a, "a")
    n, k0 = v.shape
    k = a.shape[1]
    if a.shape[0] != n:
        raise OracleError("DimensionError", f"v has {n} rows but a has {a.shape[0]}")
    if k0 + k > n:
        raise OracleError("DimensionError", f"need k0 + k <= n, got {k0}+{k} > {n}")
    if k0 == 0:
        q, r = intra(a, intra_method)
        return dict(q=q, r=r, s=np.zeros((0, k), dtype=a.dtype), kappa_t=1.0,
                    wt_inv_norm=0.0, defect=0.0)
    if k == 0:
        return dict(q=np.zeros((n, 0), dtype=a.dtype), r=np.zeros((0, 0), dtype=a.dtype),
                    s=np.zeros((k0, 0), dtype=a.dtype), kappa_t=1.0, wt_inv_norm=0.0,
                    defect=0.0)
    h = Reflector(v, choice, p)
    ah = h.apply(a, adjoint=True)                     # line 4: A <- H^* A
    s = h.p.conj().T @ ah[:k0]                         # line 5
    qb, r = intra(ah[k0:], intra_method)               # line 6
    lifted = np.zeros((n, k), dtype=qb.dtype)
    lifted[k0:] = qb
    q = h.apply(lifted)                                # line 7
    kt, wn = h.diagnostics() if diagnostics else (float("nan"), float("nan"))
    return dict(q=q, r=r, s=s, kappa_t=kt, wt_inv_norm=wn, defect=h.defect)


def block_qr(blocks, choice="qr", intra_method="householder"):
    """twostage.py:100-151 (paper Alg. 3): returns (Q, R)."""
    blocks = [to_dense(b) for b in blocks]
    n = blocks[0].shape[0]
    sizes = [b.shape[1] for b in blocks]
    tot = sum(sizes)
    rr = np.zeros((tot, tot), dtype=np.result_type(*blocks))
    q0, r0 = intra(blocks[0], intra_method)
    qs = [q0]
    rr[:sizes[0], :sizes[0]] = r0
    off = sizes[0]
    for blk, ki in zip(blocks[1:], sizes[1:]):
        res = two_stage(np.hstack(qs), blk, choice, intra_method)
        m = off
        rr[:m, off:off + ki] = res["s"]
        rr[off:off + ki, off:off + ki] = res["r"]
        qs.append(res["q"])
        off += ki
    return np.hstack(qs), rr


# ----------------------------------------------------------------------------
# B-inner product, Algorithm 4 (oblique.py)
# ----------------------------------------------------------------------------

class BInner:
    """oblique.py:36-90 for a dense HPD B, or a diagonal B given as a vector."""

    def __init__(self, b=None, diag=None):
        self.diag = None if diag is None else np.asarray(diag, dtype=np.float64)
        if b is not None:
            b = to_dense(b, "b")
            if norm2(b - b.conj().T) > 1e-12 * norm2(b):
                raise OracleError("NotHermitian", "weight matrix is not Hermitian to tolerance")
            self.b = 0.5 * (b + b.conj().T)
            self.lo = herm_chol(self.b)
        else:
            self.b = None
            self.lo_diag = np.sqrt(self.diag)

    def apply(self, x):
        return self.diag[:, None] * x if self.b is None else self.b @ x

    def lstar(self, x):                    # L^* x
        return self.lo_diag[:, None] * x if self.b is None else self.lo.conj().T @ x

    def col_norms(self, x):
        return np.sqrt((np.abs(self.lstar(x)) ** 2).sum(axis=0))

    def norm(self, x):
        m = self.lstar(x[:, None] if x.ndim == 1 else x)
        return float(np.linalg.norm(m)) if x.ndim == 1 else norm2(m)

    def defect(self, x):
        if x.size == 0:
            return 0.0
        s = np.linalg.svd(self.lstar(x), compute_uv=False)
        return float(np.max(np.abs(s ** 2 - 1.0)))

    def first_basis(self, m):
        """oblique.py:93-108 (initial_b_basis)."""
        n = self.b.shape[0] if self.b is not None else self.diag.shape[0]
        if self.b is not None:
            lm = herm_chol(self.b[:m, :m])
        else:
            lm = np.diag(np.sqrt(self.diag[:m]))
        top = trsolve(lm, np.eye(m, dtype=lm.dtype), lower=True, adjoint=True)
        u = np.zeros((n, m), dtype=lm.dtype)
        u[:m] = top
        return u


def b_house(a, u_init, inner, reorth=True, prefix=None):
    """oblique.py:170-238: left-looking B-Householder QR with one reorth."""
    a = to_dense(a)
    u_init = to_dense(u_init)
    n, k = a.shape
    dt = np.result_type(a, u_init)
    if k == 0:
        return np.zeros((n, 0), dtype=dt), np.zeros((0, 0), dtype=dt)
    thresh = 1e3 * U_ROUND * (float(inner.col_norms(a).max()) if a.size else 0.0)
    basis = u_init[:, :k].astype(dt).copy()
    r = np.zeros((k, k), dtype=dt)
    ws = np.zeros((n, k), dtype=dt)
    ts = np.zeros(k, dtype=dt)
    for j in range(k):
        y = a[:, j].astype(dt).copy()
        for i in range(j):
            y = y - ws[:, i] * ((ws[:, i].conj() @ inner.apply(y[:, None])[:, 0]) / np.conj(ts[i]))
        if j:
            c = basis[:, :j].conj().T @ inner.apply(y[:, None])[:, 0]
            r[:j, j] = c
            y = y - basis[:, :j] @ c
        beta = inner.norm(y)
        if beta <= thresh:
            raise OracleError("BreakdownError", f"column {j} is numerically zero after projection")
        y = y / beta
        al = u_init[:, j].conj() @ inner.apply(y[:, None])[:, 0]
        sg = 1.0 if al == 0 else -al / abs(al)
        basis[:, j] *= sg
        w = basis[:, j] - y
        if reorth:
            oth = basis[:, :j] if prefix is None else np.hstack([prefix, basis[:, :j]])
            if oth.size:
                w = w - oth @ (oth.conj().T @ inner.apply(w[:, None])[:, 0])
        ts[j] = w.conj() @ inner.apply(basis[:, j:j + 1])[:, 0]
        ws[:, j] = w
        r[j, j] = beta
    q = basis.copy()
    for i in range(k - 1, -1, -1):
        c = (ws[:, i].conj() @ inner.apply(q[:, i:])) / ts[i]
        q[:, i:] -= np.outer(ws[:, i], c)
    return q, np.triu(r)


def b_two_stage(v, a, u, inner, choice="qr", reorth=True, p=None, diagnostics=True):
    """oblique.py:279-315 (paper Alg. 4)."""
    v, a, u = to_dense(v), to_dense(a), to_dense(u)
    n, k0 = v.shape
    k = a.shape[1]
    if k0 == 0:
        q, r = b_house(a, u[:, :k], inner, reorth)
        return dict(q=q, r=r, s=np.zeros((0, k), dtype=a.dtype), kappa_t=1.0, wt_inv_norm=0.0)
    u0 = u[:, :k0]
    for nm, blk in (("v", v), ("u0", u0)):                        # oblique.py:141-145
        d = inner.defect(blk)
        if d > 1e-6:
            raise OracleError("OrthonormalityError", f"||{nm}^* B {nm} - I||_2 = {d:.3e}")
    coupling = v.conj().T @ inner.apply(u0)
    pm, tf = seed(coupling.conj().T, choice, p)
    x = u0 @ pm
    w = x - v
    work = a - w @ tf.solve(w.conj().T @ inner.apply(a), adjoint=True)   # H^{-1} a
    s = x.conj().T @ inner.apply(work)
    work = work - x @ s
    qb, r = b_house(work, u[:, k0:k0 + k], inner, reorth, prefix=x)
    q = qb - w @ tf.solve(w.conj().T @ inner.apply(qb))                     # H qb
    kt = wn = float("nan")
    if diagnostics:
        kt = cond_2(tf.dense())
        wn = norm2(tf.solve(w.conj().T, adjoint=True))
    return dict(q=q, r=r, s=s, kappa_t=kt, wt_inv_norm=wn)


# ----------------------------------------------------------------------------
# metrics (metrics.py:25-73) and LAPACK-sign normalisation helpers
# ----------------------------------------------------------------------------

def stability(v, a, q, r, s=None, inner=None):
    """(augmented loss ||[V,Q]^*[V,Q]-I||, cross ||V^*Q||_F, rel. residual)."""
    blk = q if v is None else np.hstack([v, q])
    if inner is not None:
        blk = inner.lstar(blk)
    sv = np.linalg.svd(blk, compute_uv=False)
    loss = float(np.max(np.abs(sv ** 2 - 1.0))) if sv.size else 0.0
    cross = 0.0
    if v is not None and v.shape[1] and q.shape[1]:
        cross = float(np.linalg.norm(v.conj().T @ (q if inner is None else inner.apply(q))))
    rec = q @ r
    if v is not None and s is not None and s.size:
        rec = rec + v @ s
    an = norm2(a)
    return loss, cross, (norm2(a - rec) / an if an > 0 else 0.0)


def gram_stability(v, a, q, r, s):
    """Gram-based (n-length-cheap) version of `stability` for large n.

    loss = max|eig([V,Q]^*[V,Q]) - 1|, residual via the Gram of the
    residual block; accurate to ~u * n, ample for the 10 n u gate."""
    vq = np.hstack([v, q]) if v is not None else q
    g = vq.conj().T @ vq
    loss = float(np.max(np.abs(np.linalg.eigvalsh(g) - 1.0)))
    res = a - q @ r - (v @ s if v is not None and s is not None and s.size else 0)
    rn = np.sqrt(max(np.linalg.eigvalsh(res.conj().T @ res).max(), 0.0))
    an = np.sqrt(max(np.linalg.eigvalsh(a.conj().T @ a).max(), 0.0))
    cross = float(np.linalg.norm(v.conj().T @ q)) if v is not None else 0.0
    return loss, cross, (rn / an if an > 0 else 0.0)
