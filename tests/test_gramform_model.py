"""CPU model of the Gram-form structured tile step that csrc/gsweep.inc (real)
and the zgs kernels of csrc/zchain.cu (complex) implement: QR([R; X]) with
reflectors v_j = [e_j; y_j] computed from the tile Gram M = X^* X alone,

    u_c = scal M[j][c],  w_c = tau (R[j][c] + u_c),  c_c = u_c - w_c yy / 2,
    M[a][b] -= conj(w_a) c_b + conj(c_a) w_b,
    Y = X Cc,  Cc = D (I + W D)^-1,  T = D_tau (I + striu(Y^* Y) D_tau)^-1,

checked here against an explicit Householder sweep on [R; X] (same LAPACK
dlarfg / zlarfg convention: beta = -sign(alpha) ||.||, alpha = R_jj real).
Host-only: this pins the algebra, the GPU parity tests pin the kernels."""
import numpy as np
import pytest


def explicit_step(r, x):
    """Householder QR of [R; X] with v_j = [e_j; y_j]: returns R', Y, taus."""
    r, x = r.copy(), x.copy()
    k = r.shape[0]
    y = np.zeros_like(x)
    taus = np.zeros(k)
    for j in range(k):
        alpha = r[j, j].real
        s2 = float(np.vdot(x[:, j], x[:, j]).real)
        if s2 == 0.0:
            continue
        beta = -np.copysign(np.sqrt(alpha * alpha + s2), alpha)
        tau = (beta - alpha) / beta
        scal = 1.0 / (alpha - beta)
        y[:, j] = scal * x[:, j]
        taus[j] = tau
        for c in range(j + 1, k):
            z = r[j, c] + np.vdot(y[:, j], x[:, c])      # v^* [R_jc; x_c]
            w = tau * z
            r[j, c] -= w
            x[:, c] -= y[:, j] * w
        r[j, j] = beta
    return r, y, taus


def gram_form_step(r, x):
    """The same step from M = X^* X only (what the kernels do)."""
    k = r.shape[0]
    r = r.copy()
    m = x.conj().T @ x
    wmat = np.zeros((k, k), dtype=r.dtype)       # W[l][c]: w_c of step l
    taus, scals = np.zeros(k), np.zeros(k)
    for j in range(k):
        alpha = r[j, j].real
        s2 = max(m[j, j].real, 0.0)
        if s2 == 0.0:
            continue
        beta = -np.copysign(np.sqrt(alpha * alpha + s2), alpha)
        tau = (beta - alpha) / beta
        scal = 1.0 / (alpha - beta)
        yy = scal * scal * s2
        u = scal * m[j, j + 1:]
        w = tau * (r[j, j + 1:] + u)
        c = u - 0.5 * yy * w
        r[j, j + 1:] -= w
        r[j, j] = beta
        wmat[j, j + 1:] = w
        m[j + 1:, j + 1:] -= np.outer(w.conj(), c) + np.outer(c.conj(), w)
        taus[j], scals[j] = tau, scal
    d = np.diag(scals)
    cc = d @ np.linalg.inv(np.eye(k) + wmat @ d)
    return r, cc, taus


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("rows,k", [(300, 12), (2048, 24)])
def test_gram_form_tile_step_matches_householder(cplx, rows, k):
    rng = np.random.default_rng(7 + rows + k + cplx)
    gen = (lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)) if cplx else (lambda *s: rng.standard_normal(s))
    head = gen(k, k)
    r0 = np.linalg.qr(head)[1]
    r0 = np.diag(np.sign(np.diag(r0).real)) @ r0 if not cplx else r0 * (np.abs(np.diag(r0)) / np.diag(r0))[:, None]
    x = gen(rows, k)
    r1, y, taus = explicit_step(r0, x)
    r2, cc, taus2 = gram_form_step(r0, x)
    scale = np.abs(r1).max()
    assert np.abs(r1 - r2).max() <= 1e-12 * scale
    assert np.abs(taus - taus2).max() <= 1e-13
    yg = x @ cc
    assert np.abs(y - yg).max() <= 1e-12 * np.abs(y).max()
    # compact WY: T = D_tau (I + striu(Y^* Y) D_tau)^-1 reproduces Q = H_1 ... H_k
    g = np.triu(yg.conj().T @ yg, 1)
    t = np.diag(taus2) @ np.linalg.inv(np.eye(k) + g @ np.diag(taus2))
    v = np.vstack([np.eye(k), yg])
    q_wy = np.eye(rows + k) - v @ t @ v.conj().T
    q_ex = np.eye(rows + k, dtype=q_wy.dtype)
    for j in range(k):
        vj = np.concatenate([np.eye(k)[:, j], y[:, j]])[:, None]
        q_ex = q_ex @ (np.eye(rows + k) - taus[j] * (vj @ vj.conj().T))
    assert np.abs(q_wy - q_ex).max() <= 1e-12
    # and the factorization itself: Q^* [R; X] = [R'; 0]
    top = q_wy.conj().T @ np.vstack([r0, x])
    assert np.abs(top[:k] - np.triu(r1)).max() <= 1e-11 * scale and np.abs(top[k:]).max() <= 1e-11 * scale
    # Q formation of the tile as the kernels do it: [C; 0] -> [C - T C; -X (Cc T C)]
    cmat = gen(k, k)
    out = q_wy @ np.vstack([cmat, np.zeros((rows, k))])
    mm = t @ cmat
    assert np.abs(out[:k] - (cmat - mm)).max() <= 1e-11 * np.abs(cmat).max()
    assert np.abs(out[k:] + x @ (cc @ mm)).max() <= 1e-11 * np.abs(out).max()


def test_direct_q_identities():
    """fastpath.cu: X^T X and V^T X per tile from the tile Grams of [V | A], and
    Q_tile = A K + V (Z1 K + Z2) = X K + V Z2 with X = A + V Z1."""
    rng = np.random.default_rng(3)
    rows, k0, k = 500, 10, 6
    v, a = rng.standard_normal((rows, k0)), rng.standard_normal((rows, k))
    z1, z2, kk = rng.standard_normal((k0, k)), rng.standard_normal((k0, k)), rng.standard_normal((k, k))
    vv, va, aa = v.T @ v, v.T @ a, a.T @ a
    x = a + v @ z1
    cx = va + vv @ z1
    assert np.abs(cx - v.T @ x).max() <= 1e-11 * np.abs(cx).max()
    mx = aa + z1.T @ cx + va.T @ z1
    assert np.abs(mx - x.T @ x).max() <= 1e-11 * np.abs(mx).max()
    q = a @ kk + v @ (z1 @ kk + z2)
    assert np.abs(q - (x @ kk + v @ z2)).max() <= 1e-11 * np.abs(q).max()
