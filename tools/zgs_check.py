"""Gram-form complex intra QR (zgs, zpath.inc) against the oracle / numpy and
the exact zchain path: parity at eligible sizes, timing of configs[3]."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(x, y, floor=1e-4):
    scale = float(np.abs(y).max())
    return float((np.abs(x - y) / (np.abs(y) + floor * scale)).max())


def parity():
    import paper_2602_14449_b200 as P
    from oracle import twostage_oracle as O
    from paper_2602_14449_b200 import _native as NT
    from paper_2602_14449_b200 import workloads as W
    rng = W.make_rng(3)
    for n, k0, k in [(1 << 20, 64, 64), (700001, 40, 48), (1 << 20, 0, 64)]:
        a = W.normal_matrix(rng, n, k) + 1j * W.normal_matrix(rng, n, k)
        if k0:
            v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0) + 1j * W.normal_matrix(rng, n, k0))
            ref = O.two_stage(v, a, "qr", diagnostics=False)
            res = P.two_stage_qr(v, a, choice="qr")
            d = {key: rel(getattr(res, key), ref[key]) for key in ("q", "r", "s")}
            m = P.compute_metrics(v, a, res)
            d["loss"], d["res"] = m.loss_orth, m.rel_residual
        else:
            q0, r0 = np.linalg.qr(a)
            res = P.householder_qr(a)
            d = {"q": rel(res.q, q0), "r": rel(res.r, r0)}
        d["fast"] = NT.last_fast(NT.context(0))
        print(f"{n}x{k0}x{k}", json.dumps(d), flush=True)


def timing():
    import torch
    import paper_2602_14449_b200 as P
    from paper_2602_14449_b200 import _native as NT
    n, k0, k = 1 << 22, 64, 64
    g = torch.Generator(device="cuda:0"); g.manual_seed(4)
    def cg(r, c):
        return torch.complex(torch.randn((r, c), generator=g, dtype=torch.float64, device="cuda:0"),
                             torch.randn((r, c), generator=g, dtype=torch.float64, device="cuda:0")) * (0.5 ** 0.5)
    v = P.householder_qr(cg(n, k0)).q.contiguous()
    a = cg(n, k)
    for _ in range(2):
        res = P.two_stage_qr(v, a)
    torch.cuda.synchronize()
    ctx = NT.context(0); L = NT.lib()
    L.ots_set_profiling(ctx, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ph = {}
    for _ in range(3):
        res = P.two_stage_qr(v, a)
        for nm, ms in NT.profile(ctx):
            ph[nm] = ph.get(nm, 0.0) + ms / 3
    e1.record(); torch.cuda.synchronize()
    L.ots_set_profiling(ctx, 0)
    m = P.compute_metrics(v, a, res, augmented=True)
    print(json.dumps({"ms": e0.elapsed_time(e1) / 3, "fast": NT.last_fast(ctx), "phases": {k_: round(v_, 3) for k_, v_ in ph.items()},
                      "loss": m.loss_orth, "res": m.rel_residual}), flush=True)


if __name__ == "__main__":
    {"parity": parity, "time": timing}[sys.argv[1] if len(sys.argv) > 1 else "parity"]()
