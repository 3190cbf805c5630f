"""Seeded synthetic inputs for the BASELINE.json configurations.

Host-side input generation only (not on the hot path).  The random streams
restate the reference's `rand.py` so that the same seed gives bit-identical
matrices to `orthoqr`:

  * make_rng       -- Philox keyed by a 64-bit seed          (rand.py:11-13)
  * standard_normal -- Box-Muller on the uniform stream       (rand.py:16-30)
  * normal_matrix  -- complex entries are (x + i y)/sqrt(2)   (rand.py:33-41)
  * uniform        -- low + (high-low) * U[0,1)              (rand.py:44-46)

The orthonormalisation of generated V blocks goes through this package's own
GPU `householder_qr` when a device is given (large n), so no host LAPACK is
needed on the bench path.
"""

from __future__ import annotations

import numpy as np


def make_rng(seed):
    return np.random.Generator(np.random.Philox(key=np.uint64(seed)))


def standard_normal(rng, shape):
    if np.isscalar(shape):
        shape = (shape,)
    count = int(np.prod(shape)) if shape else 1
    if count == 0:
        return np.zeros(shape)
    h = (count + 1) // 2
    u1 = rng.random(h)
    u2 = rng.random(h)
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    ang = (2.0 * np.pi) * u2
    out = np.empty(2 * h)
    out[:h] = rad * np.cos(ang)
    out[h:] = rad * np.sin(ang)
    return out[:count].reshape(shape)


def normal_matrix(rng, rows, cols, field="real"):
    if field == "real":
        return standard_normal(rng, (rows, cols))
    if field == "complex":
        re = standard_normal(rng, (rows, cols))
        im = standard_normal(rng, (rows, cols))
        return (re + 1j * im) / np.sqrt(2.0)
    raise ValueError(f"unknown field {field!r}")


def uniform(rng, low, high, size=None):
    return low + (high - low) * rng.random(size)


# --------------------------------------------------------------------------
# BASELINE.json configurations.  `qfactor` is injected so
# callers choose host LAPACK (tests, small n) or the GPU path (bench, big n).
# --------------------------------------------------------------------------

def config1(n=100000, k0=32, k=16, qfactor=None):
    """C1: V = Q(N(0,1) n x k0) from seed 1, A = N(0,1) n x k from seed 2."""
    qf = qfactor or _host_q
    v = qf(normal_matrix(make_rng(1), n, k0))
    a = normal_matrix(make_rng(2), n, k)
    return v, a


def config2(n=1 << 20, k0=64, k=32, qfactor=None):
    """C2: ill-conditioned A = V B + U diag(sigma) W^T, cond([V,A]) ~ 1e15."""
    qf = qfactor or _host_q
    rng = make_rng(11)
    v = qf(normal_matrix(rng, n, k0))
    bmix = normal_matrix(rng, k0, k)
    u = normal_matrix(rng, n, k)
    u = u - v @ (v.T @ u)
    u = u - v @ (v.T @ u)
    u = qf(u)
    wrot = qf(normal_matrix(rng, k, k))
    sig = np.logspace(0.0, -15.0, k)
    a = v @ bmix + (u * sig[None, :]) @ wrot.T
    return v, a


def config3(n=1 << 22, k0=128, k=64, qfactor=None):
    """C3: rank-deficient A: 32 cols in range(V), 16 random, 16 1e-30 dups."""
    qf = qfactor or _host_q
    rng = make_rng(21)
    v = qf(normal_matrix(rng, n, k0))
    a = np.empty((n, k))
    h = k // 2
    a[:, :h] = v @ normal_matrix(rng, k0, h)
    q4 = k // 4
    a[:, h:h + q4] = normal_matrix(rng, n, q4)
    a[:, h + q4:] = a[:, h:h + q4] + 1e-30 * normal_matrix(rng, n, k - h - q4)
    return v, a


def config4(n=1 << 22, k0=64, k=64, qfactor=None):
    """C4 (Euclidean part): complex Gaussian V (Q-factor) and A."""
    qf = qfactor or _host_q
    v = qf(normal_matrix(make_rng(41), n, k0, "complex"))
    a = normal_matrix(make_rng(42), n, k, "complex")
    return v, a


def config4_binner(n=1 << 22, k0=64, k=64, qfactor=None):
    """C4 (B-inner part): M = diag(d), d log-uniform on [1, 1e4);
    V M-orthonormal = D^{-1/2} Q(D^{1/2} G); u = initial_b_basis(M, k0+k)."""
    qf = qfactor or _host_q
    d = 10.0 ** uniform(make_rng(43), 0.0, 4.0, n)
    sq = np.sqrt(d)
    g = normal_matrix(make_rng(44), n, k0, "complex")
    v = qf(sq[:, None] * g) / sq[:, None]
    a = normal_matrix(make_rng(45), n, k, "complex")
    return d, v, a


def _host_q(x):
    q, _ = np.linalg.qr(x, mode="reduced")
    return q
