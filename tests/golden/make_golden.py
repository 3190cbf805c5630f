"""Generate golden fixtures by running the REAL reference package.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Each case stores its inputs and the
reference's outputs; `tests/test_oracle_golden.py` pins the oracle on them
and the GPU parity tests compare the CUDA path against them.  The file is
committed; the GPU box never needs /root/reference.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import orthoqr as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
store = {}


def put(prefix, **kw):
    for key, val in kw.items():
        store[f"{prefix}/{key}"] = np.asarray(val)


def run_two_stage(tag, v, a, choice, intra="householder", p=None):
    """Inputs are stored once per case (<case>/v, <case>/a); outputs per
    choice under <case>/<choice>/..."""
    case = tag.rsplit("/", 1)[0]
    if f"{case}/v" not in store:
        put(case, v=v, a=a)
    res = R.two_stage_qr(v, a, choice=choice, intra=intra, p=p)
    rep = R.compute_metrics(v, a, res, augmented=True)
    d = res.diagnostics
    put(tag, q=res.q, r=res.r, s=res.s, kappa_t=d.kappa_t,
        wt_inv_norm=d.wt_inv_norm, loss=rep.loss_orth, cross=rep.cross_orth,
        resid=rep.rel_residual, choice=choice, intra=intra,
        p=(p if p is not None else np.zeros((0, 0))))


def main():
    # rand.py stream pin (our workloads.py restatement must match bit-for-bit)
    rng = R.rand.make_rng(12345)
    put("rand/real", x=R.rand.normal_matrix(rng, 7, 5))
    put("rand/complex", x=R.rand.normal_matrix(R.rand.make_rng(99), 4, 3, "complex"))
    put("rand/uniform", x=R.rand.uniform(R.rand.make_rng(43), 0.0, 4.0, 9))

    # Eq. (1.2) fixture, all three choices
    v, a = R.fixture_badbcg()
    for ch in ("mlu", "qr", "polar"):
        run_two_stage(f"eq12/{ch}", v, a, ch)

    # V = [I; 0] known answer
    n, k0, k = 10, 3, 2
    v = np.zeros((n, k0)); v[:k0] = np.eye(k0)
    a = R.rand.normal_matrix(R.rand.make_rng(5), n, k)
    run_two_stage("eye/qr", v, a, "qr")

    # random real, every choice; sizes cover k0 / k not multiples of 8
    for (n, k0, k, seed) in [(200, 8, 5, 1), (333, 13, 7, 2), (1024, 32, 16, 3),
                             (768, 64, 32, 4), (520, 128, 64, 5)]:
        v = R.gen_random_orthonormal(n, k0, seed)
        a = R.rand.normal_matrix(R.rand.make_rng(seed + 100), n, k)
        for ch in ("mlu", "qr", "polar"):
            run_two_stage(f"real_{n}_{k0}_{k}/{ch}", v, a, ch)
        pexp = R.gen_random_orthonormal(k0, k0, seed + 7)
        run_two_stage(f"real_{n}_{k0}_{k}/explicit", v, a, "explicit", p=pexp)
    # cholshift intra
    v = R.gen_random_orthonormal(400, 16, 9)
    a = R.rand.normal_matrix(R.rand.make_rng(109), 400, 8)
    run_two_stage("cholshift/qr", v, a, "qr", intra="cholshift")

    # random complex
    for (n, k0, k, seed) in [(150, 6, 4, 11), (400, 32, 32, 12)]:
        v = R.gen_random_orthonormal(n, k0, seed, "complex")
        a = R.rand.normal_matrix(R.rand.make_rng(seed + 100), n, k, "complex")
        for ch in ("mlu", "qr", "polar"):
            run_two_stage(f"cplx_{n}_{k0}_{k}/{ch}", v, a, ch)

    # ill-conditioned and rank-deficient (metrics only)
    n, k0, k = 512, 16, 16
    v = R.gen_random_orthonormal(n, k0, 21)
    a = np.empty((n, k))
    a[:, :8] = v @ R.rand.normal_matrix(R.rand.make_rng(22), k0, 8)
    a[:, 8:12] = R.rand.normal_matrix(R.rand.make_rng(23), n, 4)
    a[:, 12:] = a[:, 8:12] + 1e-30 * R.rand.normal_matrix(R.rand.make_rng(24), n, 4)
    for ch in ("mlu", "qr", "polar"):
        run_two_stage(f"rankdef/{ch}", v, a, ch)

    # degenerate shapes (twostage.py:81-89)
    v = R.gen_random_orthonormal(50, 4, 31)
    a = R.rand.normal_matrix(R.rand.make_rng(32), 50, 3)
    res = R.two_stage_qr(np.zeros((50, 0)), a)
    put("k0zero", a=a, q=res.q, r=res.r, s=res.s)
    res = R.two_stage_qr(v, np.zeros((50, 0)))
    put("kzero", v=v, q=res.q, r=res.r, s=res.s)

    # householder_qr (core.py:61-84) incl. SPEC.md:42-44
    x = R.rand.normal_matrix(R.rand.make_rng(41), 300, 12)
    for nn in (False, True):
        qr = R.householder_qr(x, nonneg_diag=nn)
        put(f"hqr/nonneg{int(nn)}", a=x, q=qr.q, r=qr.r)
    qr = R.householder_qr(np.array([[3.0], [4.0]]))
    put("hqr/pyth", q=qr.q, r=qr.r)
    xc = R.rand.normal_matrix(R.rand.make_rng(42), 90, 6, "complex")
    qr = R.householder_qr(xc)
    put("hqr/complex", a=xc, q=qr.q, r=qr.r)

    # modified LU + random contraction
    z = R.rand.normal_matrix(R.rand.make_rng(51), 9, 9)
    z = z / (1.01 * np.linalg.norm(z, 2))
    for tag, zz in (("zero", np.zeros((3, 3))), ("diag", np.diag([0.5, -0.5])), ("rand", z)):
        m = R.modified_lu(zz)
        put(f"mlu/{tag}", z=zz, p=m.p_diag, l=m.l, u=m.u_tri)

    # build_reflector pieces (P, W top, T) for each choice on a random V
    v = R.gen_random_orthonormal(120, 10, 61)
    for ch in ("mlu", "qr", "polar"):
        h = R.build_reflector(v, ch)
        d = R.reflector_diagnostics(h)
        put(f"refl/{ch}", v=v, p=h.p, wtop=h.w[:10], t=h.t_solver.reconstruct(),
            kappa_t=d.kappa_t, wt_inv_norm=d.wt_inv_norm)

    # B-inner Algorithm 4: dense SPD B and a diagonal B (dense in the ref)
    n, k0, k = 120, 6, 5
    b = R.gen_spd(n, 1e3, 71)
    ip = R.InnerProduct.weighted(b)
    u = R.initial_b_basis(ip, k0 + k)
    g = R.rand.normal_matrix(R.rand.make_rng(72), n, k0)
    lt = ip.chol_b.conj().T
    vq = np.linalg.solve(lt, np.linalg.qr(lt @ g)[0])      # B-orthonormal V
    a = R.rand.normal_matrix(R.rand.make_rng(73), n, k)
    for ch in ("mlu", "qr", "polar"):
        res = R.b_two_stage_qr(vq, a, u, ip, choice=ch)
        put(f"binner_dense/{ch}", b=b, v=vq, a=a, u=u, q=res.q, r=res.r, s=res.s,
            kappa_t=res.diagnostics.kappa_t, wt_inv_norm=res.diagnostics.wt_inv_norm)
    for field in ("real", "complex"):
        n, k0, k = 256, 8, 8
        d = 10.0 ** R.rand.uniform(R.rand.make_rng(81), 0.0, 4.0, n)
        ip = R.InnerProduct.weighted(np.diag(d))
        u = R.initial_b_basis(ip, k0 + k)
        sq = np.sqrt(d)
        g = R.rand.normal_matrix(R.rand.make_rng(82), n, k0, field)
        vq = np.linalg.qr(sq[:, None] * g)[0] / sq[:, None]
        a = R.rand.normal_matrix(R.rand.make_rng(83), n, k, field)
        for ch in ("mlu", "qr", "polar"):
            res = R.b_two_stage_qr(vq, a, u, ip, choice=ch)
            put(f"binner_diag_{field}/{ch}", d=d, v=vq, a=a, u=u, q=res.q, r=res.r,
                s=res.s, kappa_t=res.diagnostics.kappa_t,
                wt_inv_norm=res.diagnostics.wt_inv_norm)

    # Algorithm 3 driver (twostage.py:100-151)
    blocks = [R.rand.normal_matrix(R.rand.make_rng(90 + i), 300, 6) for i in range(4)]
    res = R.block_householder_qr(blocks, choice="qr")
    put("block", a=np.hstack(blocks), q=res.q, r=res.r)

    # error behaviour (validation order, errors.py)
    vbad = R.gen_random_orthonormal(60, 5, 101) * 1.001
    try:
        R.two_stage_qr(vbad, np.ones((60, 2)))
    except R.OrthonormalityError as exc:
        put("err/orth", v=vbad, msg=str(exc))
    try:
        R.modified_lu(np.eye(3) * 1.5)
    except R.NormBoundError as exc:
        put("err/normbound", msg=str(exc))

    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
