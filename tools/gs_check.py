"""Gram-form level-0 factor (gsweep) vs the register-tile kernel and the
oracle: parity on assorted shapes, fallback on ill-conditioned inputs, and
timing of the headline call with OTS_GSWEEP=0 and per tall-tile height
OTS_GS_B (argv; each mode in a fresh process: the switches are read once)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parity():
    import paper_2602_14449_b200 as P
    from oracle import twostage_oracle as O
    from paper_2602_14449_b200 import workloads as W
    out = {}
    cases = [(1 << 16, 64, 64, "real"), (1 << 16, 128, 64, "real"), (1 << 16, 32, 64, "real"), (100003, 32, 48, "real"), (50000, 128, 64, "real"), (3000, 16, 40, "real"),
             (1 << 18, 128, 64, "real")]
    for n, k0, k, _ in cases:
        rng = W.make_rng(n + k0 + k)
        v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
        a = W.normal_matrix(rng, n, k)
        ref = O.two_stage(v, a, "qr")
        try:
            res = P.two_stage_qr(v, a, choice="qr")
        except Exception as exc:   # noqa: BLE001
            out[f"{n}x{k0}x{k}"] = repr(exc)
            continue
        rel = lambda x, y: float((np.abs(x - y) / (np.abs(y) + 1e-4 * np.abs(y).max())).max())
        out[f"{n}x{k0}x{k}"] = {key: rel(getattr(res, key), ref[key]) for key in ("q", "r", "s")}
    # ill-conditioned (fallback): configs[1]-like at small n
    rng = W.make_rng(7)
    n, k0, k = 1 << 16, 64, 64
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    u, _ = np.linalg.qr(W.normal_matrix(rng, n, k) - v @ (v.T @ W.normal_matrix(rng, n, k)))
    a = v @ W.normal_matrix(rng, k0, k) + (u * np.logspace(0, -15, k)) @ np.linalg.qr(W.normal_matrix(rng, k, k))[0]
    try:
        res = P.two_stage_qr(v, a, choice="qr")
    except Exception as exc:   # noqa: BLE001
        out["illcond"] = repr(exc)
        return out
    m = P.compute_metrics(v, a, res)
    out["illcond"] = {"loss": m.loss_orth, "res": m.rel_residual}
    return out


def timing():
    import torch
    import paper_2602_14449_b200 as P
    n, k0, k = 1 << 24, 128, 64
    sys.path.insert(0, ROOT)
    from bench import make_inputs
    v, a = make_inputs(n, k0, k, 0)
    for _ in range(3):
        P.two_stage_qr(v, a, choice="qr")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        res = P.two_stage_qr(v, a, choice="qr")
    e1.record()
    torch.cuda.synchronize()
    from paper_2602_14449_b200 import _native as NT
    ctx = NT.context(0)
    NT.lib().ots_set_profiling(ctx, 1)
    P.two_stage_qr(v, a, choice="qr")
    phases = NT.profile(ctx)
    NT.lib().ots_set_profiling(ctx, 0)
    vq = torch.cat([v, res.q], 1)
    from paper_2602_14449_b200.core import orthonormality_defect
    return {"ms": e0.elapsed_time(e1) / 5, "loss": orthonormality_defect(vq), "phases": phases}


if __name__ == "__main__":
    if sys.argv[1:] == ["child-parity"]:
        print(json.dumps(parity()))
    elif sys.argv[1:] == ["child-time"]:
        print(json.dumps(timing()))
    else:
        res = {}
        modes = [("gs0", {"OTS_GSWEEP": "0"}, ("parity", "time"))]
        for b in sys.argv[1:] or ["1024"]:
            modes.append((f"b{b}", {"OTS_GSWEEP": "1", "OTS_GS_B": b}, ("parity", "time")))
        for tag, extra, whats in modes:
            env = dict(os.environ, **extra)
            for what in whats:
                r = subprocess.run([sys.executable, __file__, "child-" + what], env=env, capture_output=True, text=True)
                res[f"{what}_{tag}"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else \
                    {"rc": r.returncode, "err": r.stderr[-2000:]}
                print(tag, what, json.dumps(res[f"{what}_{tag}"]), flush=True)
        print(json.dumps(res, indent=1))
