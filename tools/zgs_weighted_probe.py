"""Complex B-inner (diagonal weights) parity against the oracle at a size the
Gram-form intra QR is eligible for, exact path vs OTS_ZGS_B=1."""
import json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(x, y, floor=1e-4):
    return float((np.abs(x - y) / (np.abs(y) + floor * np.abs(y).max())).max())


def one():
    import paper_2602_14449_b200 as P
    from oracle import twostage_oracle as O
    from paper_2602_14449_b200 import _native as NT
    from paper_2602_14449_b200 import workloads as W
    out = {}
    for n, k0, k in [(560000, 64, 64), (560000, 16, 48)]:
        rng = W.make_rng(29 + k0)
        cg = lambda r, c: (W.normal_matrix(rng, r, c) + 1j * W.normal_matrix(rng, r, c)) * np.sqrt(0.5)
        d = 10.0 ** W.uniform(W.make_rng(30), 0.0, 4.0, n)
        sq = np.sqrt(d)
        v = np.linalg.qr(sq[:, None] * cg(n, k0))[0] / sq[:, None]
        a = cg(n, k)
        ip = P.InnerProduct.weighted(d)
        u = P.initial_b_basis(ip, k0 + k)
        res = P.b_two_stage_qr(v, a, u, ip)
        ref = O.b_two_stage(v, a, u, O.BInner(diag=d), "qr", diagnostics=False)
        out[f"{n}x{k0}x{k}"] = {"q": rel(res.q, ref["q"]), "r": rel(res.r, ref["r"]), "s": rel(res.s, ref["s"]),
                                "fast": NT.last_fast(NT.context(0))}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one()
    else:
        for f in ("0", "1"):
            e = dict(os.environ); e["OTS_ZGS_B"] = f
            r = subprocess.run([sys.executable, __file__, "one"], env=e, capture_output=True, text=True)
            print("OTS_ZGS_B=" + f, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:], flush=True)
