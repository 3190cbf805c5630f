"""GPU parity for complex128 (BASELINE configs[3]): two_stage_qr and
householder_qr on c128 data through the C-ABI (ots_two_stage_c128 /
ots_householder_qr_c128) against the reference's golden outputs and the CPU
oracle.  Tolerances as in test_gpu_parity.py (north_star)."""
import numpy as np
import pytest

import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O

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


def golden_cases(golden, prefix):
    keys = sorted({k.rsplit("/", 1)[0] for k in golden.files if k.endswith("/q")})
    return [k for k in keys if k.startswith(prefix)]


def cgauss(rng, n, m):
    return (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) / np.sqrt(2.0)


def test_complex_two_stage_golden(golden):
    cases = golden_cases(golden, "cplx_")
    assert cases
    for case in cases:
        base = case.rsplit("/", 1)[0]
        v, a = golden[base + "/v"], golden[base + "/a"]
        ch = str(golden[case + "/choice"])
        p = golden[case + "/p"]
        res = P.two_stage_qr(v, a, choice=ch, p=(p if p.size else None))
        assert np.iscomplexobj(res.q) and np.iscomplexobj(res.r)
        assert rel(res.q, golden[case + "/q"]) < 1e-10, case
        assert rel(res.r, golden[case + "/r"]) < 1e-10, case
        assert rel(res.s, golden[case + "/s"]) < 1e-10, case
        kt = float(golden[case + "/kappa_t"])
        wn = float(golden[case + "/wt_inv_norm"])
        assert abs(res.diagnostics.kappa_t - kt) <= 1e-10 * kt, case
        assert abs(res.diagnostics.wt_inv_norm - wn) <= 1e-10 * wn, case
        assert np.all(np.tril(res.r, -1) == 0.0)
        assert np.all(np.diag(res.r).imag == 0.0)


@pytest.mark.parametrize("choice", ["qr", "mlu", "polar", "explicit"])
def test_complex_two_stage_oracle(choice):
    rng = np.random.default_rng(7)
    n, k0, k = 6000, 32, 24
    v, _ = np.linalg.qr(cgauss(rng, n, k0))
    a = cgauss(rng, n, k)
    p = None
    if choice == "explicit":
        p, _ = np.linalg.qr(cgauss(rng, k0, k0))
    ref = O.two_stage(v, a, choice, p=p)
    res = P.two_stage_qr(v, a, choice=choice, p=p)
    assert rel(res.q, ref["q"]) < 1e-10
    assert rel(res.r, ref["r"]) < 1e-10
    assert rel(res.s, ref["s"]) < 1e-10
    assert abs(res.diagnostics.kappa_t - ref["kappa_t"]) <= 1e-10 * ref["kappa_t"]
    assert abs(res.diagnostics.wt_inv_norm - ref["wt_inv_norm"]) <= 1e-10 * ref["wt_inv_norm"]


@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (130, 64), (4099, 17), (20000, 64), (300000, 32)])
def test_complex_householder_qr(shape):
    rng = np.random.default_rng(shape[0] + shape[1])
    a = cgauss(rng, *shape)
    q0, r0 = np.linalg.qr(a)
    res = P.householder_qr(a)
    assert rel(res.r, r0) < 1e-10
    assert rel(res.q, q0) < 1e-10
    nn = P.householder_qr(a, nonneg_diag=True)
    d = np.diag(nn.r)
    assert np.all(d.imag == 0.0) and np.all(d.real >= 0.0)
    assert float(np.abs(nn.q @ nn.r - a).max() / np.abs(a).max()) < 1e-13


def test_complex_config4_like_torch():
    """configs[3] shape class on the device (n = 2^20, k0 = k = 64) with
    torch CUDA inputs; size-independent properties (loss, cross, residual)."""
    import torch
    g = torch.Generator(device="cuda:0")
    g.manual_seed(3)
    n, k0, k = 1 << 20, 64, 64
    re = torch.randn((n, k0), generator=g, dtype=torch.float64, device="cuda:0")
    im = torch.randn((n, k0), generator=g, dtype=torch.float64, device="cuda:0")
    v0 = torch.complex(re, im) / np.sqrt(2.0)
    vq = P.householder_qr(v0).q
    a = torch.complex(torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda:0"),
                      torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda:0")) / np.sqrt(2.0)
    for ch in ("qr", "mlu", "polar"):
        res = P.two_stage_qr(vq, a, choice=ch)
        Qf = torch.cat([vq, res.q], dim=1)
        G = Qf.conj().T @ Qf
        loss = torch.linalg.matrix_norm(G - torch.eye(k0 + k, dtype=G.dtype, device=G.device), ord=2).item()
        resid = (torch.linalg.matrix_norm(a - vq @ res.s - res.q @ res.r) /
                 torch.linalg.matrix_norm(a)).item()
        assert loss <= 10 * n * U, (ch, loss)
        assert resid <= 10 * n * U, (ch, resid)
        assert torch.all(torch.diagonal(res.r).imag == 0)


@pytest.mark.parametrize("ch", ["qr", "mlu", "polar"])
def test_complex_binner_diag_golden(golden, ch):
    """configs[3]'s non-standard inner product (M = diag(d)) on c128 data
    against the reference's outputs (oblique.py:279-315)."""
    g = lambda key: golden[f"binner_diag_complex/{ch}/{key}"]
    v, a = g("v"), g("a")
    ip = P.InnerProduct.weighted(np.diag(g("d")))
    u = P.initial_b_basis(ip, v.shape[1] + a.shape[1])
    assert np.array_equal(u, g("u"))
    res = P.b_two_stage_qr(v, a, u, ip, choice=ch)
    assert rel(res.q, g("q")) < 1e-10
    assert rel(res.r, g("r")) < 1e-10
    assert rel(res.s, g("s")) < 1e-10
    assert np.all(np.diag(res.r).real > 0) and np.all(np.diag(res.r).imag == 0)
    assert abs(res.diagnostics.kappa_t - float(g("kappa_t"))) < 1e-10 * float(g("kappa_t"))
    assert abs(res.diagnostics.wt_inv_norm - float(g("wt_inv_norm"))) < 1e-10 * float(g("wt_inv_norm"))


def test_complex_binner_diag_config4_like():
    """configs[3] B-inner shape class: d log-uniform in [1, 1e4], V
    M-orthonormal, complex Gaussian A; B-orthogonality and residual."""
    rng = np.random.default_rng(11)
    n, k0, k = 1 << 16, 64, 64
    d = 10.0 ** rng.uniform(0.0, 4.0, n)
    sq = np.sqrt(d)
    v = np.linalg.qr(sq[:, None] * cgauss(rng, n, k0))[0] / sq[:, None]
    a = cgauss(rng, n, k)
    ip = P.InnerProduct.weighted(d)
    u = P.initial_b_basis(ip, k0 + k)
    res = P.b_two_stage_qr(v, a, u, ip)
    ref = O.b_two_stage(v, a, u, O.BInner(diag=d), "qr", diagnostics=False)
    assert rel(res.q, ref["q"]) < 1e-10 and rel(res.r, ref["r"]) < 1e-10 and rel(res.s, ref["s"]) < 1e-10
    W = np.hstack([v, res.q])
    G = W.conj().T @ (d[:, None] * W)
    assert np.abs(G - np.eye(k0 + k)).max() <= 10 * n * U


@pytest.mark.parametrize("shape", [(500, 8), (20000, 48), (100000, 64)])
def test_complex_shifted_cholesky_qr(shape):
    """core.py:177-202 on c128 (shifted CholeskyQR + 2 refinements)."""
    rng = np.random.default_rng(shape[1])
    a = cgauss(rng, *shape)
    q0, r0 = O.cholqr_shifted(a)
    res = P.shifted_cholesky_qr(a)
    assert rel(res.r, r0) < 1e-10
    assert rel(res.q, q0) < 1e-10
    assert np.all(np.diag(res.r).real > 0)


def test_complex_shifted_cholesky_breakdown():
    a = np.zeros((100, 4), dtype=np.complex128)
    a[:, 0] = 1.0
    with pytest.raises(P.NotPositiveDefinite):
        P.shifted_cholesky_qr(a)


@pytest.mark.parametrize("choice", ["qr", "mlu"])
def test_complex_two_stage_cholshift_oracle(choice):
    rng = np.random.default_rng(17)
    n, k0, k = 8000, 24, 16
    v, _ = np.linalg.qr(cgauss(rng, n, k0))
    a = cgauss(rng, n, k)
    ref = O.two_stage(v, a, choice, intra_method="cholshift")
    res = P.two_stage_qr(v, a, choice=choice, intra="cholshift")
    assert rel(res.q, ref["q"]) < 1e-10
    assert rel(res.r, ref["r"]) < 1e-10
    assert rel(res.s, ref["s"]) < 1e-10


@pytest.mark.parametrize("n", [1, 5, 40])
def test_complex_modified_lu(n):
    rng = np.random.default_rng(n)
    z = np.linalg.qr(cgauss(rng, 2 * n, n))[0][:n]   # ||z|| <= 1
    p0, l0, u0 = O.mlu(z)
    res = P.modified_lu(z)
    assert np.array_equal(np.asarray(res.p_diag), p0)
    assert rel(res.l, l0) < 1e-12 and rel(res.u_tri, u0) < 1e-12


def test_complex_b_householder_and_block_driver():
    """b_householder_qr / b_block_householder_qr (oblique.py:170-238, 318-361)
    on c128 blocks with M = diag(d), against the oracle block by block."""
    rng = np.random.default_rng(23)
    n, sizes = 900, [16, 24, 16]
    d = 10.0 ** rng.uniform(0.0, 2.0, n)
    ip, ref_in = P.InnerProduct.weighted(d), O.BInner(diag=d)
    a = cgauss(rng, n, sum(sizes))
    u = P.initial_b_basis(ip, sum(sizes))
    r1 = P.b_householder_qr(a[:, :16], u[:, :16], ip)
    q1, rr1 = O.b_house(a[:, :16], u[:, :16], ref_in)
    assert rel(r1.q, q1) < 1e-10 and rel(r1.r, rr1) < 1e-10
    blocks = [a[:, sum(sizes[:i]):sum(sizes[:i + 1])] for i in range(len(sizes))]
    res = P.b_block_householder_qr(blocks, ip)
    qs, off = [q1], sizes[0]
    rf = np.zeros((sum(sizes), sum(sizes)), dtype=complex)
    rf[:16, :16] = rr1
    for i in range(1, len(sizes)):
        out = O.b_two_stage(np.hstack(qs), blocks[i], u[:, :off + sizes[i]], ref_in, "qr", diagnostics=False)
        qs.append(out["q"])
        rf[:off, off:off + sizes[i]] = out["s"]
        rf[off:off + sizes[i], off:off + sizes[i]] = out["r"]
        off += sizes[i]
    assert np.iscomplexobj(res.q)
    assert rel(res.q, np.hstack(qs)) < 1e-10 and rel(res.r, rf) < 1e-10
