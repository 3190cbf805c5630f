"""Full-size BASELINE.json configurations on one GPU: device time of each call
(CUDA events, inputs resident, 1 warm-up + median of 3) and the stability
metrics of its result from the GPU metrics judge (compute_metrics, augmented
[V, Q]: loss ||[V,Q]^*[V,Q] - I||_2, relative residual), against 10 n u.

Inputs are the seeded generators of `workloads.py` (the reference's rand.py
streams); V blocks are orthonormalised with this package's GPU QR.  The
Krylov sweep (configs[4]) builds A <- L Q_prev (1D Laplacian) with torch
element-wise ops (input generation, not the measured path).

    python tools/configs_report.py [--out profiles/r01e_configs.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_14449_b200 as P  # noqa: E402
from paper_2602_14449_b200 import workloads as W  # noqa: E402

U = 2.0 ** -53


def gpu_q(x):
    return P.householder_qr(torch.from_numpy(np.ascontiguousarray(x)).cuda()).q.cpu().numpy()


def gpu_qb(x):   # > 64 columns: block Householder QR in 64-column blocks
    g = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return P.block_householder_qr([g[:, i:i + 64].contiguous() for i in range(0, g.shape[1], 64)]).q.cpu().numpy()


def f_alg(n, k0, k, cf=1):
    return cf * (8.0 * n * k0 * k + 4.0 * (n - k0) * k * k - 4.0 / 3.0 * k ** 3 + n * k0 * (k0 + 1.0))


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], out


def metrics(v, a, res, inner=None):
    """GPU metrics judge (compute_metrics, augmented [V, Q], real or complex)."""
    m = P.compute_metrics(v, a, res, inner=inner, augmented=True)
    return float(m.loss_orth), float(m.rel_residual)


def entry(name, n, k0, k, ms, res, v, a, cf=1, inner=None, extra=None):
    loss, resid = metrics(v, a, res, inner)
    e = {"config": name, "n": n, "k0": k0, "k": k, "ms": round(ms, 3),
         "gflops": round(f_alg(n, k0, k, cf) / (ms * 1e-3) / 1e9, 1),
         "loss": loss, "residual": resid, "bound_10nu": 10 * n * U,
         "kappa_t": res.diagnostics.kappa_t, "wt_inv_norm": res.diagnostics.wt_inv_norm}
    if extra:
        e.update(extra)
    print(json.dumps(e), flush=True)
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip5", action="store_true")
    args = ap.parse_args()
    out = []
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()

    v, a = W.config1(qfactor=gpu_q)
    V, A = dev(v), dev(a)
    ms, res = timed(lambda: P.two_stage_qr(V, A))
    out.append(entry("C1 well-conditioned", v.shape[0], v.shape[1], a.shape[1], ms, res, V, A))

    v, a = W.config2(qfactor=gpu_q)
    V, A = dev(v), dev(a)
    for ch in ("qr", "mlu", "polar"):
        ms, res = timed(lambda: P.two_stage_qr(V, A, choice=ch))
        out.append(entry(f"C2 ill-conditioned ({ch})", v.shape[0], v.shape[1], a.shape[1], ms, res, V, A))
    del V, A

    v, a = W.config3(qfactor=gpu_qb)
    V, A = dev(v), dev(a)
    for ch in ("qr", "mlu", "polar"):
        ms, res = timed(lambda: P.two_stage_qr(V, A, choice=ch))
        out.append(entry(f"C3 rank-deficient ({ch})", v.shape[0], v.shape[1], a.shape[1], ms, res, V, A))
    del V, A, v, a

    cq = lambda x: P.householder_qr(torch.from_numpy(np.ascontiguousarray(x)).cuda()).q.cpu().numpy()
    v, a = W.config4(qfactor=cq)
    V, A = dev(v), dev(a)
    ms, res = timed(lambda: P.two_stage_qr(V, A))
    out.append(entry("C4 complex128", v.shape[0], v.shape[1], a.shape[1], ms, res, V, A, cf=4))
    del V, A, v, a
    d, v, a = W.config4_binner(qfactor=cq)
    ip = P.InnerProduct.weighted(dev(d))
    V, A = dev(v), dev(a)
    u = P.initial_b_basis(ip, v.shape[1] + a.shape[1])
    ms, res = timed(lambda: P.b_two_stage_qr(V, A, u, ip))
    out.append(entry("C4 complex128 B-inner M=diag(d)", v.shape[0], v.shape[1], a.shape[1], ms, res, V, A, cf=4,
                     inner=ip))
    del V, A, v, a, u

    if not args.skip5:   # configs[4]: block-Krylov sweep, n = 2^24, k = 64, k0 = 0, 64, ..., 512
        n, k = 1 << 24, 64
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        A0 = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda")
        kb = P.KrylovBasis(n, 9 * k, device=0, incremental_gram=True)
        kb.append(A0)
        del A0
        torch.cuda.empty_cache()
        for step in range(1, 9):
            k0 = step * k
            qprev = kb.q[:, k0 - k:k0]
            Lq = 2.0 * qprev
            Lq[1:] -= qprev[:-1]
            Lq[:-1] -= qprev[1:]
            Vv = kb.q[:, :k0]
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = kb.append(Lq)
            e1.record()
            torch.cuda.synchronize()
            out.append(entry(f"C5 Krylov step {step} (KrylovBasis, incremental Gram)", n, k0, k,
                             e0.elapsed_time(e1), res, Vv, Lq))
            del Lq, res
            torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
