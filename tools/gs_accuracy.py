"""Per-entry parity of the Gram-form level-0 factor against the oracle on the
B-inner (diagonal weight) case of tests/test_gpu_parity.py, per tall-tile
height OTS_GS_B and with OTS_GSWEEP=0 (each mode in a fresh process: the
switches are read once)."""
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


def one():
    import paper_2602_14449_b200 as P
    from oracle import twostage_oracle as O
    from paper_2602_14449_b200 import workloads as W
    out = {}
    n, k0, k = 1 << 18, 64, 64
    d = 10.0 ** W.uniform(W.make_rng(43), 0.0, 4.0, n)
    sq = np.sqrt(d)
    v = np.linalg.qr(sq[:, None] * W.normal_matrix(W.make_rng(44), n, k0))[0] / sq[:, None]
    a = W.normal_matrix(W.make_rng(45), n, k)
    ip = P.InnerProduct.weighted(d)
    u = P.initial_b_basis(ip, k0 + k)
    res = P.b_two_stage_qr(v, a, u, ip)
    ref = O.b_two_stage(v, a, u, O.BInner(diag=d), "qr", diagnostics=False)
    out["binner"] = {key: rel(getattr(res, key), ref[key]) for key in ("q", "r", "s")}
    # the same rows through the Euclidean call (scaled problem)
    vs, as_ = sq[:, None] * v, sq[:, None] * a
    res = P.two_stage_qr(vs, as_, choice="qr")
    ref = O.two_stage(vs, as_, "qr")
    out["scaled_euclid"] = {key: rel(getattr(res, key), ref[key]) for key in ("q", "r", "s")}
    # plain Gaussian at the same shape
    v2, _ = np.linalg.qr(W.normal_matrix(W.make_rng(46), n, k0))
    res = P.two_stage_qr(v2, a, choice="qr")
    ref = O.two_stage(v2, a, "qr")
    out["gauss"] = {key: rel(getattr(res, key), ref[key]) for key in ("q", "r", "s")}
    # intra QR alone vs LAPACK
    qr = P.householder_qr(as_)
    q0, r0 = np.linalg.qr(as_)
    out["hqr_scaled"] = {"q": rel(qr.q, q0), "r": rel(qr.r, r0)}
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        print(json.dumps(one()))
        sys.exit(0)
    allout = {}
    for name, env in [("gsweep0", {"OTS_GSWEEP": "0"}), ("b256", {"OTS_GS_B": "256"}), ("b512", {"OTS_GS_B": "512"}),
                      ("b1024", {"OTS_GS_B": "1024"}), ("b2048", {})]:
        e = dict(os.environ)
        e.update(env)
        r = subprocess.run([sys.executable, __file__, "one"], env=e, capture_output=True, text=True)
        try:
            allout[name] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:   # noqa: BLE001
            allout[name] = r.stderr[-400:]
        print(name, json.dumps(allout[name]), flush=True)
