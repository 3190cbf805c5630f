"""GPU parity of the direct-Q pipeline (csrc/fastpath.cu: tile Grams of
[V | A], no materialised X) against the CPU oracle on the same seeded inputs,
its fall-back to the materialised-X pipeline on inputs that cancel, and the
reference's error behaviour on shapes that take it (twostage.py:57-97).
Tolerances as in test_gpu_parity.py (BASELINE.json north_star)."""
import numpy as np
import pytest

import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O
from paper_2602_14449_b200 import _native as NT
from paper_2602_14449_b200 import workloads as W

from .test_gpu_parity import rel

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def took_fast():
    return NT.last_fast(NT.context(0))


@pytest.mark.parametrize("n,k0,k,choice", [(1 << 20, 128, 64, "qr"), (600001, 100, 48, "mlu"),
                                           (560000, 128, 33, "polar"), (600000, 97, 64, "qr")])
def test_direct_q_vs_oracle(n, k0, k, choice):
    rng = W.make_rng(n + k0 + k)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    ref = O.two_stage(v, a, choice, diagnostics=True)
    res = P.two_stage_qr(v, a, choice=choice)
    assert took_fast() == 1
    assert rel(res.q, ref["q"]) < 1e-10
    assert rel(res.r, ref["r"]) < 1e-10
    assert rel(res.s, ref["s"]) < 1e-10
    assert np.all(np.tril(res.r, -1) == 0.0)
    assert abs(res.diagnostics.kappa_t - ref["kappa_t"]) <= 1e-10 * ref["kappa_t"]
    assert abs(res.diagnostics.wt_inv_norm - ref["wt_inv_norm"]) <= 1e-10 * ref["wt_inv_norm"]


def test_direct_q_device_tensors():
    import torch
    n, k0, k = 560000, 128, 64
    rng = W.make_rng(5)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    ref = O.two_stage(v, a, "qr", diagnostics=False)
    res = P.two_stage_qr(torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda())
    assert took_fast() == 1
    assert rel(res.q.cpu().numpy(), ref["q"]) < 1e-10
    assert rel(res.r.cpu().numpy(), ref["r"]) < 1e-10
    assert rel(res.s.cpu().numpy(), ref["s"]) < 1e-10


def _metrics_ok(v, a, res, ref):
    """loss, residual <= 10 n u and <= 10x the oracle's own (Gram-based judge)"""
    n = v.shape[0]
    loss, _, resid = O.gram_stability(v, a, res.q, res.r, res.s)
    rl, _, rr = O.gram_stability(v, a, ref["q"], ref["r"], ref["s"])
    assert loss <= 10 * n * U and resid <= 10 * n * U
    assert loss <= 10 * max(rl, 4 * U) and resid <= 10 * max(rr, 4 * U)


def test_direct_q_falls_back_on_rank_deficient():
    # configs[2]-like: the first columns of A lie in range(V), so X = H^* A
    # cancels and the tile Grams of [V | A] cannot carry X^T X
    n, k0, k = 560000, 128, 64
    rng = W.make_rng(7)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    a[:, :32] = v @ W.normal_matrix(rng, k0, 32)
    a[:, 40:44] = a[:, 36:40] + 1e-30 * W.normal_matrix(rng, n, 4)
    ref = O.two_stage(v, a, "qr", diagnostics=False)
    res = P.two_stage_qr(v, a, choice="qr")
    assert took_fast() == 0
    _metrics_ok(v, a, res, ref)


def test_direct_q_falls_back_on_ill_conditioned():
    # configs[1]-like: A = V B + U diag(sigma) W^T, sigma down to 1e-15
    n, k0, k = 560000, 128, 64
    rng = W.make_rng(11)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    g = W.normal_matrix(rng, n, k)
    u, _ = np.linalg.qr(g - v @ (v.T @ g))
    w, _ = np.linalg.qr(W.normal_matrix(rng, k, k))
    a = v @ W.normal_matrix(rng, k0, k) + (u * np.logspace(0, -15, k)) @ w.T
    ref = O.two_stage(v, a, "qr", diagnostics=False)
    res = P.two_stage_qr(v, a, choice="qr")
    assert took_fast() == 0
    _metrics_ok(v, a, res, ref)


def test_direct_q_shape_errors_and_non_finite():
    n, k0, k = 560000, 128, 64
    rng = W.make_rng(13)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    bad = v.copy()
    bad[:, 3] *= 1.0 + 1e-6
    with pytest.raises(P.OrthonormalityError):
        P.two_stage_qr(bad, a)
    an = a.copy()
    an[n // 2, 5] = np.nan
    with pytest.raises(ValueError):
        P.two_stage_qr(v, an)
    ai = a.copy()
    ai[17, 0] = np.inf
    with pytest.raises(ValueError):
        P.two_stage_qr(v, ai)
    # and a clean call on the same context afterwards
    res = P.two_stage_qr(v, a)
    assert took_fast() == 1
    m = P.compute_metrics(v, a, res)
    assert m.loss_orth <= 10 * n * U and m.rel_residual <= 10 * n * U


def test_direct_q_inside_the_block_driver():
    """Alg. 3 driver (twostage.py:100-151): the block that meets a 128-column
    basis takes the direct-Q pipeline; Q, R as the oracle's.  With the
    incremental Gram (a Krylov-type caller) the call keeps the materialised-X
    pipeline."""
    import torch
    n = 560000
    rng = W.make_rng(91)
    blocks = [W.normal_matrix(rng, n, 64) for _ in range(3)]
    rq, rr = O.block_qr(blocks, "qr")
    res = P.block_householder_qr(blocks)
    assert took_fast() == 1
    assert rel(res.q, rq) < 1e-10 and rel(res.r, rr) < 1e-10
    kb = P.KrylovBasis(n, 192, device=0, incremental_gram=True)
    for b in blocks:
        kb.append(torch.from_numpy(b).cuda())
    assert took_fast() == 0
    assert rel(kb.q.cpu().numpy(), rq) < 1e-10


# ---------------------------------------------------------------------------
# complex128: Gram-form intra QR on tall tiles (zgs, csrc/zchain.cu + zpath.inc)
# ---------------------------------------------------------------------------
def _cgauss(rng, n, k):
    return (W.normal_matrix(rng, n, k) + 1j * W.normal_matrix(rng, n, k)) * np.sqrt(0.5)


@pytest.mark.parametrize("n,k0,k,choice", [(1 << 20, 64, 64, "qr"), (600001, 40, 48, "mlu"), (560000, 24, 33, "polar")])
def test_complex_gram_form_vs_oracle(n, k0, k, choice):
    rng = W.make_rng(300 + k0 + k)
    v, _ = np.linalg.qr(_cgauss(rng, n, k0))
    a = _cgauss(rng, n, k)
    ref = O.two_stage(v, a, choice, diagnostics=True)
    res = P.two_stage_qr(v, a, choice=choice)
    assert took_fast() == 1
    assert rel(res.q, ref["q"]) < 1e-10
    assert rel(res.r, ref["r"]) < 1e-10
    assert rel(res.s, ref["s"]) < 1e-10
    assert np.all(np.tril(res.r, -1) == 0.0) and np.abs(np.diag(res.r).imag).max() == 0.0
    assert abs(res.diagnostics.kappa_t - ref["kappa_t"]) <= 1e-10 * ref["kappa_t"]


def test_complex_gram_form_householder_qr():
    n, k = 560000, 64
    a = _cgauss(W.make_rng(21), n, k)
    q0, r0 = np.linalg.qr(a)
    res = P.householder_qr(a)
    assert took_fast() == 1
    assert rel(res.q, q0) < 1e-10 and rel(res.r, r0) < 1e-10


def test_complex_gram_form_falls_back():
    # nearly dependent columns after the projection: the sweep's cancellation
    # factor flags the chains and the call takes the exact zchain path
    n, k0, k = 560000, 32, 64
    rng = W.make_rng(23)
    v, _ = np.linalg.qr(_cgauss(rng, n, k0))
    a = _cgauss(rng, n, k)
    a[:, :16] = v @ _cgauss(rng, k0, 16)
    a[:, 40:44] = a[:, 36:40] + 1e-30 * _cgauss(rng, n, 4)
    ref = O.two_stage(v, a, "qr", diagnostics=False)
    res = P.two_stage_qr(v, a)
    assert took_fast() == 0
    loss, _, resid = O.gram_stability(v, a, res.q, res.r, res.s)
    rl, _, rr = O.gram_stability(v, a, ref["q"], ref["r"], ref["s"])
    assert loss <= 10 * n * U and resid <= 10 * n * U
    assert loss <= 10 * max(rl, 4 * U) and resid <= 10 * max(rr, 4 * U)


def test_complex_weighted_rows_gram_form_vs_oracle():
    """B = diag(d), complex: the scaled Euclidean problem takes the Gram-form
    intra QR too; Q, R, S per entry against the oracle's B-path."""
    n, k0, k = 560000, 16, 48
    rng = W.make_rng(29)
    d = 10.0 ** W.uniform(W.make_rng(30), 0.0, 4.0, n)
    sq = np.sqrt(d)
    v = np.linalg.qr(sq[:, None] * _cgauss(rng, n, k0))[0] / sq[:, None]
    a = _cgauss(rng, n, k)
    ip = P.InnerProduct.weighted(d)
    u = P.initial_b_basis(ip, k0 + k)
    res = P.b_two_stage_qr(v, a, u, ip)
    assert took_fast() == 1
    ref = O.b_two_stage(v, a, u, O.BInner(diag=d), "qr", diagnostics=False)
    assert rel(res.q, ref["q"]) < 1e-10 and rel(res.r, ref["r"]) < 1e-10 and rel(res.s, ref["s"]) < 1e-10
    m = P.compute_metrics(v, a, res, inner=ip)
    assert m.loss_orth <= 10 * n * U and m.rel_residual <= 10 * n * U
