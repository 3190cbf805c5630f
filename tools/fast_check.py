"""Direct-Q pipeline (fastpath.cu) against the oracle and the materialised-X
pipeline: parity on eligible shapes, fallback on ill-conditioned inputs,
phase times at the headline (argv: parity | time)."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(x, y, floor=1e-4):
    scale = float(np.abs(y).max())
    return float((np.abs(x - y) / (np.abs(y) + floor * scale)).max())


def last_fast():
    from paper_2602_14449_b200 import _native as NT
    L = NT.lib()
    L.ots_last_fast.argtypes = [C.c_void_p]
    return int(L.ots_last_fast(NT.context(0)))


def parity():
    import paper_2602_14449_b200 as P
    from oracle import twostage_oracle as O
    from paper_2602_14449_b200 import workloads as W
    out = {}
    for n, k0, k in [(1 << 20, 128, 64), (700001, 100, 48), (1 << 20, 128, 33), (1 << 22, 128, 64), (3000000, 97, 64)]:
        rng = W.make_rng(n + k0 + k)
        v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
        a = W.normal_matrix(rng, n, k)
        ref = O.two_stage(v, a, "qr", diagnostics=False)
        res = P.two_stage_qr(v, a, choice="qr")
        d = {key: rel(getattr(res, key), ref[key]) for key in ("q", "r", "s")}
        d["fast"] = last_fast()
        m = P.compute_metrics(v, a, res)
        d["loss"], d["res"] = m.loss_orth, m.rel_residual
        out[f"{n}x{k0}x{k}"] = d
        print(f"{n}x{k0}x{k}", json.dumps(d), flush=True)
    # rank-deficient / ill-conditioned: must fall back
    rng = W.make_rng(7)
    n, k0, k = 1 << 20, 128, 64
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    a[:, :32] = v @ W.normal_matrix(rng, k0, 32)
    res = P.two_stage_qr(v, a, choice="qr")
    m = P.compute_metrics(v, a, res)
    out["rankdef"] = {"fast": last_fast(), "loss": m.loss_orth, "res": m.rel_residual}
    print("rankdef", json.dumps(out["rankdef"]), flush=True)
    return out


def timing():
    import torch
    import paper_2602_14449_b200 as P
    from paper_2602_14449_b200 import _native as NT
    from bench import make_inputs
    n, k0, k = int(os.environ.get("FC_N", 1 << 24)), 128, 64
    v, a = make_inputs(n, k0, k, 0)
    for _ in range(3):
        res = P.two_stage_qr(v, a, choice="qr")
    torch.cuda.synchronize()
    ctx = NT.context(0)
    L = NT.lib()
    L.ots_set_profiling(ctx, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ph = {}
    for _ in range(5):
        res = P.two_stage_qr(v, a, choice="qr")
        for nm, ms in NT.profile(ctx):
            ph[nm] = ph.get(nm, 0.0) + ms / 5
    e1.record()
    torch.cuda.synchronize()
    L.ots_set_profiling(ctx, 0)
    m = P.compute_metrics(v, a, res, augmented=True)
    print(json.dumps({"ms": e0.elapsed_time(e1) / 5, "fast": last_fast(), "phases": ph, "loss": m.loss_orth,
                      "res": m.rel_residual}), flush=True)


def sizes():
    """ms per call, fast on / off, per n (each mode in a fresh process)"""
    import subprocess
    for fast in ("1", "0"):
        e = dict(os.environ)
        e["OTS_FAST"] = fast
        r = subprocess.run([sys.executable, __file__, "sizes1"], env=e, capture_output=True, text=True)
        print("OTS_FAST=" + fast, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:], flush=True)


def sizes1():
    import torch
    import paper_2602_14449_b200 as P
    from bench import make_inputs
    out = {}
    for n in (1 << 19, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
        v, a = make_inputs(n, 128, 64, 0)
        for _ in range(3):
            P.two_stage_qr(v, a, choice="qr")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.two_stage_qr(v, a, choice="qr")
        e1.record()
        torch.cuda.synchronize()
        out[n] = [round(e0.elapsed_time(e1) / 5, 3), last_fast()]
        del v, a
    print(json.dumps(out))


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
    {"parity": parity, "time": timing, "sizes": sizes, "sizes1": sizes1}[mode]()
