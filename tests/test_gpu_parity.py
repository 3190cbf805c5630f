"""GPU parity: the CUDA path (through the C-ABI, via the drop-in facade)
against the reference's golden outputs and the CPU oracle on the same seeded
inputs.  Tolerances (BASELINE.json north_star):
  * elementwise Q, R, S within 1e-10 relative on well-conditioned inputs
    (same LAPACK sign convention), kappa_t / wt_inv_norm within 1e-10 rel;
  * loss of orthogonality and relative residual <= 10 n u and <= 10x the
    oracle's own values on ill-conditioned / rank-deficient inputs.
"""
import numpy as np
import pytest

import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O
from paper_2602_14449_b200 import workloads as W

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def rel(x, y, floor=1e-4):
    """Elementwise relative difference with an absolute floor of
    floor * max|y| for entries at the roundoff scale of the block."""
    x, y = np.asarray(x), np.asarray(y)
    if y.size == 0:
        return 0.0
    scale = max(float(np.abs(y).max()), 1e-300)
    return float((np.abs(x - y) / (np.abs(y) + floor * scale)).max())


def nrel(x, y):
    """normwise max|x - y| / max|y| (for residual checks)"""
    x, y = np.asarray(x), np.asarray(y)
    return float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-300)) if y.size else 0.0


def golden_cases(golden, prefix):
    keys = sorted({k.rsplit("/", 1)[0] for k in golden.files if k.endswith("/q")})
    return [k for k in keys if k.startswith(prefix)]


@pytest.mark.parametrize("group", ["eq12", "eye", "real_"])
def test_two_stage_golden(golden, group):
    cases = golden_cases(golden, group)
    assert cases
    for case in cases:
        base = case.rsplit("/", 1)[0]
        v, a = golden[base + "/v"], golden[base + "/a"]
        ch = str(golden[case + "/choice"])
        p = golden[case + "/p"]
        res = P.two_stage_qr(v, a, choice=ch, p=(p if p.size else None))
        # Eq.(1.2): R = diag(1e-30, 1e-30) -- compare absolutely at its own scale
        assert rel(res.q, golden[case + "/q"]) < 1e-10, case
        assert rel(res.r, golden[case + "/r"]) < 1e-10, case
        assert rel(res.s, golden[case + "/s"]) < 1e-10, case
        kt = float(golden[case + "/kappa_t"])
        wn = float(golden[case + "/wt_inv_norm"])
        assert abs(res.diagnostics.kappa_t - kt) <= 1e-10 * kt, case
        assert abs(res.diagnostics.wt_inv_norm - wn) <= 1e-10 * wn, case
        assert np.all(np.tril(res.r, -1) == 0.0)


def test_rankdef_metrics(golden):
    for case in golden_cases(golden, "rankdef"):
        v, a = golden["rankdef/v"], golden["rankdef/a"]
        ch = str(golden[case + "/choice"])
        res = P.two_stage_qr(v, a, choice=ch)
        loss, cross, resid = O.stability(v, a, res.q, res.r, res.s)
        n = v.shape[0]
        assert loss <= 10 * n * U and resid <= 10 * n * U
        assert loss <= 10 * max(float(golden[case + "/loss"]), 4 * U)
        assert resid <= 10 * max(float(golden[case + "/resid"]), 4 * U)


def test_householder_qr_golden(golden):
    for nn in (0, 1):
        qr = P.householder_qr(golden[f"hqr/nonneg{nn}/a"], nonneg_diag=bool(nn))
        assert rel(qr.q, golden[f"hqr/nonneg{nn}/q"]) < 1e-10
        assert rel(qr.r, golden[f"hqr/nonneg{nn}/r"]) < 1e-10
    qr = P.householder_qr(np.array([[3.0], [4.0]]))          # SPEC.md:43 (LAPACK signs)
    assert np.allclose(qr.q[:, 0], [-0.6, -0.8]) and np.isclose(qr.r[0, 0], -5.0)
    qr = P.householder_qr(np.array([[3.0], [4.0]]), nonneg_diag=True)
    assert np.allclose(qr.q[:, 0], [0.6, 0.8]) and np.isclose(qr.r[0, 0], 5.0)
    qr = P.householder_qr(np.eye(3))
    assert np.allclose(qr.q, np.eye(3)) and np.allclose(qr.r, np.eye(3))


def test_modified_lu_golden(golden):
    for tag in ("zero", "diag", "rand"):
        m = P.modified_lu(golden[f"mlu/{tag}/z"])
        assert np.array_equal(m.p_diag, golden[f"mlu/{tag}/p"])
        assert rel(m.l, golden[f"mlu/{tag}/l"]) < 1e-12
        assert rel(m.u_tri, golden[f"mlu/{tag}/u"]) < 1e-12
    with pytest.raises(P.NormBoundError):
        P.modified_lu(np.eye(3) * 1.5)


def test_errors(golden):
    with pytest.raises(P.OrthonormalityError) as ei:
        P.two_stage_qr(golden["err/orth/v"], np.ones((60, 2)))
    assert str(ei.value) == str(golden["err/orth/msg"])
    with pytest.raises(P.DimensionError):
        P.two_stage_qr(np.eye(5, 3), np.ones((5, 3)))
    with pytest.raises(P.ParameterError):
        P.two_stage_qr(np.eye(8, 2), np.ones((8, 2)), choice="nope")
    with pytest.raises(ValueError):
        a = np.ones((8, 2)); a[3, 1] = np.nan
        P.two_stage_qr(np.eye(8, 2), a)


def test_degenerate(golden):
    res = P.two_stage_qr(np.zeros((50, 0)), golden["k0zero/a"])
    assert rel(res.q, golden["k0zero/q"]) < 1e-10 and res.s.shape == (0, 3)
    res = P.two_stage_qr(golden["kzero/v"], np.zeros((50, 0)))
    assert res.q.shape == (50, 0) and res.s.shape == (4, 0)


@pytest.mark.parametrize("n,k0,k", [(1 << 14, 32, 16), (1 << 16, 64, 32), (1 << 17, 128, 64),
                                    (40000, 13, 7), (5000, 100, 50)])
@pytest.mark.parametrize("choice", ["qr", "mlu", "polar"])
def test_vs_oracle_random(n, k0, k, choice):
    rng = W.make_rng(1000 + n + k0)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    ref = O.two_stage(v, a, choice, diagnostics=(n <= 1 << 16))
    res = P.two_stage_qr(v, a, choice=choice)
    assert rel(res.q, ref["q"]) < 1e-10
    assert rel(res.r, ref["r"]) < 1e-10
    assert rel(res.s, ref["s"]) < 1e-10
    if n <= 1 << 16:
        assert abs(res.diagnostics.kappa_t - ref["kappa_t"]) <= 1e-10 * ref["kappa_t"]
        assert abs(res.diagnostics.wt_inv_norm - ref["wt_inv_norm"]) <= 1e-10 * ref["wt_inv_norm"]


def test_config2_like_illconditioned():
    v, a = W.config2(n=1 << 16, k0=64, k=32)
    res = P.two_stage_qr(v, a)
    loss, cross, resid = O.gram_stability(v, a, res.q, res.r, res.s)
    ref = O.two_stage(v, a, "qr", diagnostics=False)
    rl, rc, rr = O.gram_stability(v, a, ref["q"], ref["r"], ref["s"])
    n = v.shape[0]
    assert loss <= 10 * n * U and resid <= 10 * n * U
    assert loss <= 10 * max(rl, 4 * U) and resid <= 10 * max(rr, 4 * U)


def test_config3_like_rankdef():
    v, a = W.config3(n=1 << 16, k0=128, k=64)
    for ch in ("qr", "mlu", "polar"):
        res = P.two_stage_qr(v, a, choice=ch)
        loss, cross, resid = O.gram_stability(v, a, res.q, res.r, res.s)
        n = v.shape[0]
        assert loss <= 10 * n * U and resid <= 10 * n * U, ch


def test_cholshift_golden(golden):
    v, a = golden["cholshift/v"], golden["cholshift/a"]
    res = P.two_stage_qr(v, a, choice="qr", intra="cholshift")
    assert rel(res.q, golden["cholshift/qr/q"]) < 1e-10
    assert rel(res.r, golden["cholshift/qr/r"]) < 1e-10
    assert rel(res.s, golden["cholshift/qr/s"]) < 1e-10


def test_shifted_cholesky_qr_vs_oracle():
    rng = W.make_rng(321)
    x = W.normal_matrix(rng, 50000, 24)
    qr = P.shifted_cholesky_qr(x)
    q, r = O.cholqr_shifted(x)
    assert rel(qr.q, q) < 1e-10 and rel(qr.r, r) < 1e-10


def test_cholshift_breakdown_is_intra_failure():
    # exactly rank-deficient remainder: Cholesky of the shifted Gram may pass,
    # but a zero column makes the refinement Gram singular -> IntraFailure
    n = 4000
    v = np.zeros((n, 2)); v[0, 0] = v[1, 1] = 1.0
    a = np.zeros((n, 3)); a[5:, 0] = 1.0   # columns 1, 2 exactly zero
    with pytest.raises((P.IntraFailure,)):
        P.two_stage_qr(v, a, intra="cholshift")


@pytest.mark.parametrize("ch", ["mlu", "qr", "polar"])
def test_binner_diag_golden(golden, ch):
    g = lambda key: golden[f"binner_diag_real/{ch}/{key}"]
    ip = P.InnerProduct.weighted(np.diag(g("d")))
    u = P.initial_b_basis(ip, 16)
    assert np.array_equal(u, g("u"))
    res = P.b_two_stage_qr(g("v"), g("a"), u, ip, choice=ch)
    assert rel(res.q, g("q")) < 1e-10
    assert rel(res.r, g("r")) < 1e-10
    assert rel(res.s, g("s")) < 1e-10
    assert np.all(np.diag(res.r) > 0)
    assert abs(res.diagnostics.kappa_t - float(g("kappa_t"))) < 1e-10 * float(g("kappa_t"))
    assert abs(res.diagnostics.wt_inv_norm - float(g("wt_inv_norm"))) < 1e-10 * float(g("wt_inv_norm"))


@pytest.mark.parametrize("ch", ["mlu", "qr", "polar"])
def test_binner_dense_golden(golden, ch):
    # dense SPD B (oblique.py:48-56): Cholesky transform on the GPU
    g = lambda key: golden[f"binner_dense/{ch}/{key}"]
    ip = P.InnerProduct.weighted(g("b"))
    k0, k = g("v").shape[1], g("a").shape[1]
    u = P.initial_b_basis(ip, k0 + k)
    assert rel(u, g("u")) < 1e-12
    res = P.b_two_stage_qr(g("v"), g("a"), g("u"), ip, choice=ch)
    assert rel(res.q, g("q")) < 1e-10
    assert rel(res.r, g("r")) < 1e-10
    assert rel(res.s, g("s")) < 1e-10
    assert np.all(np.diag(res.r) > 0)
    assert abs(res.diagnostics.kappa_t - float(g("kappa_t"))) < 1e-10 * float(g("kappa_t"))
    assert abs(res.diagnostics.wt_inv_norm - float(g("wt_inv_norm"))) < 1e-10 * float(g("wt_inv_norm"))


@pytest.mark.parametrize("n,k0,k,choice", [(700, 24, 16, "qr"), (1500, 64, 64, "mlu"), (2048, 96, 32, "polar")])
def test_binner_dense_vs_oracle(n, k0, k, choice):
    rng = W.make_rng(71 + n)
    X = W.normal_matrix(rng, n, n)
    b = X @ X.T / n + np.eye(n)                       # SPD, cond ~ 5
    ip = P.InnerProduct.weighted(b)
    ref_in = O.BInner(b=b)
    lo = np.linalg.cholesky(b)
    v = np.linalg.solve(lo.T, np.linalg.qr(W.normal_matrix(rng, n, k0))[0])   # B-orthonormal
    a = W.normal_matrix(rng, n, k)
    u = P.initial_b_basis(ip, k0 + k)
    res = P.b_two_stage_qr(v, a, u, ip, choice=choice)
    ref = O.b_two_stage(v, a, u, ref_in, choice, diagnostics=True)
    assert rel(res.q, ref["q"]) < 1e-10 and rel(res.r, ref["r"]) < 1e-10 and rel(res.s, ref["s"]) < 1e-10
    assert abs(res.diagnostics.wt_inv_norm - ref["wt_inv_norm"]) < 1e-10 * ref["wt_inv_norm"]
    # k0 = 0: B-orthonormal QR of A
    r0 = P.b_two_stage_qr(np.zeros((n, 0)), a, u, ip)
    ref0 = O.b_two_stage(np.zeros((n, 0)), a, u, ref_in, "qr", diagnostics=False)
    assert rel(r0.q, ref0["q"]) < 1e-10 and rel(r0.r, ref0["r"]) < 1e-10


def test_binner_dense_errors():
    n = 64
    b = np.eye(n); b[0, 1] = 1.0                      # not symmetric
    with pytest.raises(P.NotHermitian):
        P.InnerProduct.weighted(b)
    b = np.eye(n); b[3, 3] = -1.0; b[0, 1] = b[1, 0] = 0.1   # symmetric, indefinite
    with pytest.raises(P.NotPositiveDefinite):
        P.InnerProduct.weighted(b)
    b = np.eye(n) + 0.01 * np.ones((n, n))
    ip = P.InnerProduct.weighted(b)
    v = np.zeros((n, 2)); v[0, 0] = v[1, 1] = 1.0
    u = np.eye(n)[:, :5]                              # not the canonical basis of this B
    with pytest.raises(P.OrthonormalityError) as ei:  # v is not B-orthonormal (oblique.py:141-145)
        P.b_two_stage_qr(v, np.ones((n, 3)), u, ip)
    assert "v^* B v" in str(ei.value)


def test_binner_diag_vs_oracle_large():
    n, k0, k = 1 << 18, 64, 64
    d = 10.0 ** W.uniform(W.make_rng(43), 0.0, 4.0, n)
    sq = np.sqrt(d)
    v = np.linalg.qr(sq[:, None] * W.normal_matrix(W.make_rng(44), n, k0))[0] / sq[:, None]
    a = W.normal_matrix(W.make_rng(45), n, k)
    ip = P.InnerProduct.weighted(d)
    u = P.initial_b_basis(ip, k0 + k)
    res = P.b_two_stage_qr(v, a, u, ip)
    ref = O.b_two_stage(v, a, u, O.BInner(diag=d), "qr", diagnostics=False)
    assert rel(res.q, ref["q"]) < 1e-10 and rel(res.r, ref["r"]) < 1e-10 and rel(res.s, ref["s"]) < 1e-10


@pytest.mark.parametrize("k0,k,choice", [(200, 48, "qr"), (384, 64, "qr"), (256, 64, "mlu"),
                                         (160, 32, "polar")])
def test_large_k0_vs_oracle(k0, k, choice):
    n = 1 << 15
    rng = W.make_rng(900 + k0)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    ref = O.two_stage(v, a, choice, diagnostics=True)
    res = P.two_stage_qr(v, a, choice=choice)
    assert rel(res.q, ref["q"]) < 1e-10
    assert rel(res.r, ref["r"]) < 1e-10
    assert rel(res.s, ref["s"]) < 1e-10
    assert abs(res.diagnostics.kappa_t - ref["kappa_t"]) <= 1e-10 * ref["kappa_t"]
    assert abs(res.diagnostics.wt_inv_norm - ref["wt_inv_norm"]) <= 1e-10 * ref["wt_inv_norm"]


def test_block_krylov_sweep_small():
    """configs[4] shape at small n: k0 = 0, 64, ..., 512 with A <- L Q_prev."""
    import torch
    n, k, steps = 1 << 14, 64, 8
    a0 = W.normal_matrix(W.make_rng(5), n, k)

    def lap(q):
        out = 2.0 * q
        out[1:] -= q[:-1]
        out[:-1] -= q[1:]
        return out

    qs = [P.two_stage_qr(np.zeros((n, 0)), a0).q]
    assert rel(qs[0], O.two_stage(np.zeros((n, 0)), a0)["q"]) < 1e-10
    for i in range(steps):
        vq = np.hstack(qs)
        ai = lap(qs[-1])
        res = P.two_stage_qr(vq, ai)
        # every step elementwise against the oracle on the same inputs (the
        # sweep itself amplifies earlier roundoff through L, so the blocks of
        # two independent sweeps are not compared)
        rr = O.two_stage(vq, ai, diagnostics=False)
        assert rel(res.q, rr["q"]) < 1e-10 and rel(res.r, rr["r"]) < 1e-10 and rel(res.s, rr["s"]) < 1e-10, i
        qs.append(res.q)
    Qg = np.hstack(qs)
    loss = np.abs(np.linalg.eigvalsh(Qg.T @ Qg) - 1).max()
    assert loss <= 10 * n * U


@pytest.mark.parametrize("ch", ["mlu", "qr", "polar"])
def test_reflector_api_golden(golden, ch):
    v = golden[f"refl/{ch}/v"]
    h = P.build_reflector(v, ch)
    assert rel(h.p, golden[f"refl/{ch}/p"]) < 1e-12
    assert rel(h.w[:10], golden[f"refl/{ch}/wtop"]) < 1e-12
    assert rel(h.t_solver.reconstruct(), golden[f"refl/{ch}/t"]) < 1e-12
    d = P.reflector_diagnostics(h)
    assert abs(d.kappa_t - float(golden[f"refl/{ch}/kappa_t"])) < 1e-10 * d.kappa_t
    assert abs(d.wt_inv_norm - float(golden[f"refl/{ch}/wt_inv_norm"])) < 1e-10 * d.wt_inv_norm


@pytest.mark.parametrize("ch", ["qr", "mlu", "polar"])
def test_apply_reflector_vs_oracle(ch):
    rng = W.make_rng(55)
    n, k0, m = 20000, 48, 80
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    x = W.normal_matrix(rng, n, m)
    h = P.build_reflector(v, ch)
    ho = O.Reflector(v, ch)
    for adj in (False, True):
        assert rel(P.apply_reflector(h, x, adjoint=adj), ho.apply(x, adjoint=adj)) < 1e-10
    # v = [I;0], qr seed -> H = diag(-I, I)
    e = np.zeros((10, 3)); e[:3] = np.eye(3)
    he = P.build_reflector(e, "qr")
    assert np.allclose(P.apply_reflector(he, np.eye(10)[:, :1]), -np.eye(10)[:, :1])
    assert np.allclose(P.apply_reflector(he, np.eye(10)[:, 3:4]), np.eye(10)[:, 3:4])
    # t_solver.solve round trip
    b = W.normal_matrix(rng, k0, 5)
    tt = h.t_solver.reconstruct()
    assert nrel(tt @ h.t_solver.solve(b), b) < 1e-12
    assert nrel(tt.T @ h.t_solver.solve(b, adjoint=True), b) < 1e-12


def test_stream_front_end_matches_calls():
    """two_stage_qr_stream (host buffers, overlapped transfers) returns the
    same Q, R, S as individual two_stage_qr calls, for every call."""
    import torch
    rng = np.random.default_rng(5)
    n, k0, k = 40000, 32, 16
    pairs, refs = [], []
    for i in range(3):
        v = np.linalg.qr(rng.standard_normal((n, k0)))[0]
        a = rng.standard_normal((n, k))
        pairs.append((torch.from_numpy(v).pin_memory(), torch.from_numpy(a).pin_memory()))
        refs.append(P.two_stage_qr(v, a))
    # consume with immediate copies (output buffers rotate over two slots)
    got = []
    for r in P.two_stage_qr_stream(pairs):
        r.wait()
        got.append((r.q.numpy().copy(), r.r.numpy().copy(), r.s.numpy().copy()))
    assert len(got) == 3
    for (q, r_, s), ref in zip(got, refs):
        assert rel(q, ref.q) < 1e-13 and rel(r_, ref.r) < 1e-13 and rel(s, ref.s) < 1e-13


@pytest.mark.parametrize("case", ["small", "augmented", "illcond"])
def test_gpu_metrics_vs_oracle(case):
    """metrics.py (compute_metrics / orthogonality_loss) on the GPU against the
    oracle's SVD-based values (loss and cross absolute to 1e-13, residual to 1e-3
    relative or 1e-16 absolute)."""
    rng = np.random.default_rng(9)
    n, k0, k = 20000, 48, 24
    v = np.linalg.qr(rng.standard_normal((n, k0)))[0]
    a = rng.standard_normal((n, k))
    if case == "illcond":
        a[:, 1] = a[:, 0] + 1e-9 * a[:, 1]
    res = P.two_stage_qr(v, a)
    loss, cross, resid = O.stability(v, a, res.q, res.r, res.s)
    rep = P.compute_metrics(v, a, res, augmented=(case != "small"))
    if case == "small":
        loss = float(np.max(np.abs(np.linalg.svd(res.q, compute_uv=False) ** 2 - 1)))
    assert abs(rep.loss_orth - loss) < 1e-13
    assert abs(rep.cross_orth - cross) < 1e-13
    assert abs(rep.rel_residual - resid) <= max(1e-3 * resid, 1e-16)
    assert rep.kappa_t == res.diagnostics.kappa_t
    assert abs(P.orthogonality_loss(res.q, v=v) - O.stability(v, a, res.q, res.r, res.s)[0]) < 1e-13


def _b_case(kind, n, k0, k, seed):
    rng = W.make_rng(seed)
    if kind == "diag":
        d = 10.0 ** W.uniform(rng, 0.0, 2.0, n)
        ip, ref_in, lo = P.InnerProduct.weighted(d), O.BInner(diag=d), np.diag(np.sqrt(d))
    else:
        X = W.normal_matrix(rng, n, n)
        b = X @ X.T / n + np.eye(n)
        ip, ref_in, lo = P.InnerProduct.weighted(b), O.BInner(b=b), np.linalg.cholesky(b)
    v = np.linalg.solve(lo.T, np.linalg.qr(W.normal_matrix(rng, n, k0))[0])   # B-orthonormal
    a = W.normal_matrix(rng, n, k)
    return ip, ref_in, v, a


@pytest.mark.parametrize("kind", ["diag", "dense"])
@pytest.mark.parametrize("choice", ["mlu", "qr", "polar"])
def test_b_reflector_vs_oracle(kind, choice):
    """b_build_reflector / b_apply_reflector (oblique.py:125-161) against the
    oracle's inline B-reflector of b_two_stage (oracle/twostage_oracle.py)."""
    n, k0, k = 900, 24, 16
    ip, ref_in, v, a = _b_case(kind, n, k0, k, 300 + k0)
    u0 = P.initial_b_basis(ip, k0)
    h = P.b_build_reflector(v, u0, ip, choice=choice)
    coupling = v.T @ ref_in.apply(u0)
    pm, tf = O.seed(coupling.T, choice, None)
    x = u0 @ pm
    w = x - v
    assert rel(h.p, pm) < 1e-10 and rel(h.x, x) < 1e-10 and rel(h.w, w) < 1e-10
    hinv_a = a - w @ tf.solve(w.T @ ref_in.apply(a), adjoint=True)
    h_a = a - w @ tf.solve(w.T @ ref_in.apply(a))
    assert rel(P.b_apply_reflector(h, a, inverse=True), hinv_a) < 1e-10
    assert rel(P.b_apply_reflector(h, a), h_a) < 1e-10
    # H maps x = u0 p onto v and is B-unitary
    assert rel(P.b_apply_reflector(h, x), v) < 1e-10
    y = P.b_apply_reflector(h, a)
    assert rel(y.T @ ref_in.apply(y), a.T @ ref_in.apply(a)) < 1e-10
    ts = h.t_solver.solve(np.eye(k0))
    assert rel(ts, tf.solve(np.eye(k0))) < 1e-10
    with pytest.raises(P.OrthonormalityError):
        P.b_build_reflector(2.0 * v, u0, ip, choice=choice)
    with pytest.raises(P.DimensionError):
        P.b_build_reflector(v[:, :3], u0, ip)


@pytest.mark.parametrize("kind", ["diag", "dense"])
def test_b_householder_qr_vs_oracle(kind):
    n, k = 1100, 48
    ip, ref_in, _, a = _b_case(kind, n, 8, k, 410)
    u = P.initial_b_basis(ip, k)
    res = P.b_householder_qr(a, u, ip)
    q, r = O.b_house(a, u, ref_in)
    assert rel(res.q, q) < 1e-10 and rel(res.r, r) < 1e-10
    assert np.all(np.diag(res.r) > 0)
    # torch in -> torch out, on the device
    t = pytest.importorskip("torch")
    rt = P.b_householder_qr(t.from_numpy(a).cuda(), t.from_numpy(u).cuda(), ip)
    assert rt.q.is_cuda and rel(rt.q.cpu().numpy(), q) < 1e-10
    a0 = a.copy()
    a0[:, 5] = 0.0
    with pytest.raises(P.BreakdownError):
        P.b_householder_qr(a0, u, ip)
    assert P.b_householder_qr(np.zeros((n, 0)), u, ip).q.shape == (n, 0)


@pytest.mark.parametrize("kind", ["diag", "dense"])
def test_b_block_householder_qr_vs_oracle(kind):
    """oblique.py:318-361 against the oracle driven block by block."""
    n, sizes = 1200, [16, 24, 32]
    ip, ref_in, _, a = _b_case(kind, n, 8, sum(sizes), 520)
    blocks = [a[:, sum(sizes[:i]):sum(sizes[:i + 1])] for i in range(len(sizes))]
    res = P.b_block_householder_qr(blocks, ip)
    u = ref_in.first_basis(sum(sizes))
    q0, r0 = O.b_house(blocks[0], u[:, :sizes[0]], ref_in)
    qs, rf = [q0], np.zeros((sum(sizes), sum(sizes)))
    rf[:sizes[0], :sizes[0]] = r0
    off = sizes[0]
    for i in range(1, len(sizes)):
        qa = np.hstack(qs)
        out = O.b_two_stage(qa, blocks[i], u[:, :off + sizes[i]], ref_in, "qr", diagnostics=False)
        qs.append(out["q"])
        rf[:off, off:off + sizes[i]] = out["s"]
        rf[off:off + sizes[i], off:off + sizes[i]] = out["r"]
        off += sizes[i]
    assert rel(res.q, np.hstack(qs)) < 1e-10 and rel(res.r, rf) < 1e-10
    assert res.block_sizes == sizes
    assert nrel(res.q @ res.r, a) < 1e-12
    bad = [b.copy() for b in blocks]
    bad[0][:, 3] = 0.0
    with pytest.raises(P.IntraFailure) as ei:
        P.b_block_householder_qr(bad, ip)
    assert ei.value.block == 0


@pytest.mark.parametrize("kind", ["diag", "dense"])
def test_b_householder_qr_general_basis(kind):
    """Any B-orthonormal u_init: the positive-diagonal B-QR is unique, so the
    result matches the reference run with that same u_init."""
    n, k = 800, 24
    ip, ref_in, _, a = _b_case(kind, n, 8, k, 610)
    lo = np.diag(np.sqrt(ref_in.diag)) if kind == "diag" else np.linalg.cholesky(ref_in.b)
    u = np.linalg.solve(lo.T, np.linalg.qr(W.normal_matrix(W.make_rng(611), n, k))[0])
    res = P.b_householder_qr(a, u, ip)
    q, r = O.b_house(a, u, ref_in)
    assert rel(res.q, q) < 1e-10 and rel(res.r, r) < 1e-10
    m = P.compute_metrics(None, a, res, inner=ip)
    assert m.loss_orth < 1e-13 and m.rel_residual < 1e-14
    with pytest.raises(NotImplementedError):
        P.b_householder_qr(a, 2.0 * u, ip)


def test_apply_reflector_complex_rhs():
    """A real reflector applied to complex x (reflector.py:231-238 with numpy
    promotion): real and imaginary parts independently."""
    n, k0 = 600, 12
    rng = W.make_rng(77)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    h = P.build_reflector(v)
    x = W.normal_matrix(rng, n, 5) + 1j * W.normal_matrix(rng, n, 5)
    for adj in (False, True):
        y = P.apply_reflector(h, x, adjoint=adj)
        assert np.iscomplexobj(y)
        assert rel(y.real, P.apply_reflector(h, x.real.copy(), adjoint=adj)) < 1e-15
        assert rel(y.imag, P.apply_reflector(h, x.imag.copy(), adjoint=adj)) < 1e-15
    b = x[:k0]
    z = h.t_solver.solve(b, adjoint=True)
    assert np.iscomplexobj(z) and rel(z.imag, h.t_solver.solve(b.imag.copy(), adjoint=True)) < 1e-15
