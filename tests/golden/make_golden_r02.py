"""Round-2 golden fixtures, made by running the REAL reference package.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_r02.py

Writes tests/golden/golden_r02.npz (committed; the GPU box never reads the
reference).  Cases: the Alg. 3 / Krylov drivers (block_householder_qr real
and complex, reorthogonalized_two_stage with sweeps=2 and the bcgs sequence),
the baselines (bcgs_two_stage, bcgs2_block Euclidean / diagonal-B / dense-B,
bmgs_inter plain and WY, cholqr_two_stage), shifted_cholesky_qr with other
refinement counts, complex compute_metrics, InnerProduct's
apply/gram/col_norms/norm/defect, the validation order of two_stage_qr /
build_reflector, and the paper's Table-4 shape (n=1000, k0=k=100).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import orthoqr as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_r02.npz")
store = {}


def put(prefix, **kw):
    for key, val in kw.items():
        store[f"{prefix}/{key}"] = np.asarray(val)


def err_of(fn):
    try:
        fn()
    except Exception as exc:   # noqa: BLE001 -- the class name is the fixture
        return type(exc).__name__, str(exc)
    return "none", ""


def main():
    nm, rng = R.rand.normal_matrix, R.rand.make_rng

    # --- Algorithm 3 driver (twostage.py:100-151), complex blocks
    blocks = [nm(rng(190 + i), 240, 5, "complex") for i in range(3)]
    res = R.block_householder_qr(blocks, choice="qr")
    put("blockc", a=np.hstack(blocks), q=res.q, r=res.r, kappa=res.diagnostics.kappa_t)
    blocks = [nm(rng(290 + i), 500, 8) for i in range(5)]
    for ch in ("mlu", "polar"):
        res = R.block_householder_qr(blocks, choice=ch)
        put(f"blockr/{ch}", a=np.hstack(blocks), q=res.q, r=res.r, kappa=res.diagnostics.kappa_t)

    # --- reorthogonalized_two_stage (twostage.py:154-180)
    for fld, tag in (("real", "r"), ("complex", "c")):
        v = R.gen_random_orthonormal(400, 12, 7, fld)
        a = nm(rng(8), 400, 6, fld)
        res = R.reorthogonalized_two_stage(v, a, "qr", sweeps=2)
        put(f"reorth_{tag}", v=v, a=a, q=res.q, r=res.r, s=res.s, hist=np.array(res.sweep_history))
        seq = ["inter", "intra", "inter", "intra"]
        res = R.reorthogonalized_two_stage(v, a, "bcgs", sequence=seq)
        put(f"bcgs_{tag}", q=res.q, r=res.r, s=res.s, hist=np.array(res.sweep_history))
        res = R.cholqr_two_stage(v, a)
        put(f"cholqr_{tag}", q=res.q, r=res.r, s=res.s)
        put(f"bmgs_{tag}", plain=R.bmgs_inter([v[:, :5], v[:, 5:]], a),
            wy=R.bmgs_inter([v[:, :5], v[:, 5:9], v[:, 9:]], a, wy=True))
        res = R.bcgs_two_stage(v, a, ["inter", "intra"], intra="cholshift")
        put(f"bcgs1chol_{tag}", q=res.q, r=res.r, s=res.s, hist=np.array(res.sweep_history))

    # --- bcgs2_block (baselines.py:76-125): Euclidean, diagonal B, dense B
    blocks = [nm(rng(390 + i), 200, 4) for i in range(3)]
    res = R.bcgs2_block(blocks)
    put("bcgs2/euc", a=np.hstack(blocks), q=res.q, r=res.r)
    d = 10.0 ** R.rand.uniform(rng(43), 0.0, 2.0, 200)
    ipd = R.InnerProduct.weighted(np.diag(d))
    res = R.bcgs2_block(blocks, inner=ipd)
    put("bcgs2/diag", d=d, q=res.q, r=res.r)
    b = R.gen_spd(200, 1e3, 17)
    ipb = R.InnerProduct.weighted(b)
    res = R.bcgs2_block(blocks, inner=ipb, intra="cholshift")
    put("bcgs2/dense", b=b, q=res.q, r=res.r)

    # --- InnerProduct methods (oblique.py:62-90)
    x = nm(rng(501), 200, 5)
    y = nm(rng(502), 200, 3)
    for tag, ip in (("diag", ipd), ("dense", ipb)):
        put(f"ip/{tag}", x=x, y=y, apply=ip.apply(x), gram=ip.gram(x, y), col_norms=ip.col_norms(x),
            norm=ip.norm(x), norm1=ip.norm(x[:, 0]), defect=ip.defect(x))

    # --- shifted_cholesky_qr refinement counts (core.py:177-202)
    a = nm(rng(601), 300, 7)
    for rp in (0, 1, 3):
        qr = R.shifted_cholesky_qr(a, refine_passes=rp)
        put(f"chol/{rp}", a=a, q=qr.q, r=qr.r)

    # --- complex metrics (metrics.py:25-73)
    v = R.gen_random_orthonormal(500, 10, 31, "complex")
    a = nm(rng(32), 500, 6, "complex")
    res = R.two_stage_qr(v, a)
    res.q = res.q + 1e-9 * nm(rng(33), 500, 6, "complex")     # non-trivial loss and residual
    rep = R.compute_metrics(v, a, res, augmented=True)
    put("zmetrics", v=v, a=a, q=res.q, r=res.r, s=res.s, loss=rep.loss_orth, cross=rep.cross_orth,
        resid=rep.rel_residual, loss_q=R.metrics.orthogonality_loss(res.q))

    # --- validation order (errors.py; reflector.py:207-228, twostage.py:45-97)
    vbad = R.gen_random_orthonormal(60, 5, 101) * 1.001
    vok = R.gen_random_orthonormal(60, 5, 102)
    a = np.ones((60, 2))
    anan = a.copy()
    anan[3, 1] = np.nan
    cases = {
        "bad_choice_nonorth": lambda: R.two_stage_qr(vbad, a, choice="nope"),
        "bad_intra_nonorth": lambda: R.two_stage_qr(vbad, a, intra="nope"),
        "explicit_nop_nonorth": lambda: R.two_stage_qr(vbad, a, choice="explicit"),
        "explicit_badshape_nonorth": lambda: R.two_stage_qr(vbad, a, choice="explicit", p=np.eye(3)),
        "bad_choice_ok": lambda: R.two_stage_qr(vok, a, choice="nope"),
        "bad_intra_ok": lambda: R.two_stage_qr(vok, a, intra="nope"),
        "bad_intra_nan": lambda: R.two_stage_qr(vok, anan, intra="nope"),
        "nan_ok": lambda: R.two_stage_qr(vok, anan),
        "explicit_badshape_ok": lambda: R.two_stage_qr(vok, a, choice="explicit", p=np.eye(3)),
        "refl_bad_choice_nonorth": lambda: R.build_reflector(vbad, choice="nope"),
        "refl_bad_choice_allow": lambda: R.build_reflector(vbad, choice="nope", allow_defect=True),
        "k0zero_bad_intra": lambda: R.two_stage_qr(np.zeros((60, 0)), a, intra="nope"),
        "k0zero_bad_choice": lambda: R.two_stage_qr(np.zeros((60, 0)), a, choice="nope"),
    }
    put("order", vbad=vbad, vok=vok)
    for key, fn in cases.items():
        cls, msg = err_of(fn)
        put(f"order/{key}", cls=cls, msg=msg)
    put("order/k0zero_bad_choice_q", q=R.two_stage_qr(np.zeros((60, 0)), nm(rng(7), 60, 2), choice="nope").q)

    # --- the paper's Table-4 shape: n=1000, k0=k=100
    v = R.gen_random_orthonormal(1000, 100, 1)
    a = nm(rng(40010), 1000, 100)
    for ch in ("mlu", "qr", "polar"):
        res = R.two_stage_qr(v, a, choice=ch)
        put(f"table4/{ch}", q=res.q, r=res.r, s=res.s, kappa_t=res.diagnostics.kappa_t,
            wt_inv_norm=res.diagnostics.wt_inv_norm)
    put("table4", v=v, a=a)

    # --- complex reflector objects (reflector.py:156-247)
    v = R.gen_random_orthonormal(300, 9, 61, "complex")
    x = nm(rng(62), 300, 5, "complex")
    b = nm(rng(63), 9, 4, "complex")
    put("zrefl", v=v, x=x, b=b)
    for ch in ("mlu", "qr", "polar"):
        h = R.build_reflector(v, ch)
        d = R.reflector_diagnostics(h)
        put(f"zrefl/{ch}", p=h.p, t=h.t_solver.reconstruct(), w=h.w, hx=R.apply_reflector(h, x),
            hhx=R.apply_reflector(h, x, adjoint=True), sol=h.t_solver.solve(b),
            sola=h.t_solver.solve(b, adjoint=True), kappa_t=d.kappa_t, wt_inv_norm=d.wt_inv_norm)

    # --- wide complex two_stage (k > 64)
    v = R.gen_random_orthonormal(700, 20, 71, "complex")
    a = nm(rng(72), 700, 80, "complex")
    res = R.two_stage_qr(v, a)
    put("zwide", v=v, a=a, q=res.q, r=res.r, s=res.s, kappa_t=res.diagnostics.kappa_t,
        wt_inv_norm=res.diagnostics.wt_inv_norm)

    # --- B-path with a general (non-canonical) B-orthonormal basis u
    n, k0, k = 400, 6, 5
    for fld, tag in (("real", "r"), ("complex", "c")):
        d = 10.0 ** R.rand.uniform(rng(81), 0.0, 2.0, n)
        ip = R.InnerProduct.weighted(np.diag(d))
        sq = np.sqrt(d)[:, None]
        v = np.linalg.qr(sq * nm(rng(82), n, k0, fld))[0] / sq
        u = np.linalg.qr(sq * nm(rng(83), n, k0 + k, fld))[0] / sq
        a = nm(rng(84), n, k, fld)
        x = nm(rng(85), n, 3, fld)
        put(f"bgen_{tag}", d=d, v=v, u=u, a=a, x=x)
        for ch in ("mlu", "qr", "polar"):
            res = R.b_two_stage_qr(v, a, u, ip, choice=ch)
            h = R.b_build_reflector(v, u[:, :k0], ip, choice=ch)
            dg = R.oblique.b_reflector_diagnostics(h)
            put(f"bgen_{tag}/{ch}", q=res.q, r=res.r, s=res.s, kappa_t=res.diagnostics.kappa_t,
                wt_inv_norm=res.diagnostics.wt_inv_norm, p=h.p, t=h.t_solver.reconstruct(), w=h.w, hx=h.x,
                ax=R.b_apply_reflector(h, x), aix=R.b_apply_reflector(h, x, inverse=True),
                dk=dg.kappa_t, dw=dg.wt_inv_norm)
    b = R.gen_spd(n, 1e2, 87)
    ipb = R.InnerProduct.weighted(b)
    lt = np.linalg.cholesky(b).T
    v = np.linalg.solve(lt, np.linalg.qr(nm(rng(88), n, k0))[0])
    u = np.linalg.solve(lt, np.linalg.qr(nm(rng(89), n, k0 + k))[0])
    a = nm(rng(90), n, k)
    res = R.b_two_stage_qr(v, a, u, ipb, choice="qr")
    put("bgen_dense", b=b, v=v, u=u, a=a, q=res.q, r=res.r, s=res.s, kappa_t=res.diagnostics.kappa_t,
        wt_inv_norm=res.diagnostics.wt_inv_norm)
    ipe = R.InnerProduct.euclidean()
    v = R.gen_random_orthonormal(n, k0, 91)
    u = R.gen_random_orthonormal(n, k0 + k, 92)
    res = R.b_two_stage_qr(v, a, u, ipe, choice="mlu")
    put("bgen_euc", v=v, u=u, a=a, q=res.q, r=res.r, s=res.s, kappa_t=res.diagnostics.kappa_t,
        wt_inv_norm=res.diagnostics.wt_inv_norm)

    # --- dense complex Hermitian B (oblique.py:36-361 with a complex weight)
    n, k0, k = 240, 6, 5
    uu = np.linalg.qr(nm(rng(101), n, n, "complex"))[0]
    b = (uu * (10.0 ** np.linspace(0.0, 2.0, n))) @ uu.conj().T
    ipz = R.InnerProduct.weighted(b)
    lh = ipz.chol_b.conj().T
    v = np.linalg.solve(lh, np.linalg.qr(nm(rng(102), n, k0, "complex"))[0])
    ucan = R.initial_b_basis(ipz, k0 + k)
    ugen = np.linalg.solve(lh, np.linalg.qr(nm(rng(103), n, k0 + k, "complex"))[0])
    a = nm(rng(104), n, k, "complex")
    x = nm(rng(105), n, 3, "complex")
    xr = nm(rng(106), n, 2)
    put("zdense", b=b, v=v, ucan=ucan, ugen=ugen, a=a, x=x, xr=xr, apply=ipz.apply(x), gram=ipz.gram(x, v),
        col_norms=ipz.col_norms(x), norm=ipz.norm(x), defect=ipz.defect(v), apply_r=ipz.apply(xr))
    for ch in ("mlu", "qr", "polar"):
        for tag, u in (("can", ucan), ("gen", ugen)):
            res = R.b_two_stage_qr(v, a, u, ipz, choice=ch)
            h = R.b_build_reflector(v, u[:, :k0], ipz, choice=ch)
            put(f"zdense/{ch}_{tag}", q=res.q, r=res.r, s=res.s, kappa_t=res.diagnostics.kappa_t,
                wt_inv_norm=res.diagnostics.wt_inv_norm, p=h.p, w=h.w, ax=R.b_apply_reflector(h, x),
                aix=R.b_apply_reflector(h, x, inverse=True))
    qr = R.b_householder_qr(a, ucan[:, :k], ipz)
    put("zdense/bhqr", q=qr.q, r=qr.r)
    blocks = [nm(rng(107 + i), n, 4, "complex") for i in range(3)]
    res = R.b_block_householder_qr(blocks, ipz, choice="qr")
    put("zdense/bblock", b0=blocks[0], b1=blocks[1], b2=blocks[2], q=res.q, r=res.r,
        kappa_t=res.diagnostics.kappa_t)

    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
