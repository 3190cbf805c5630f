import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O
rng = np.random.default_rng(1)
def cg(n, m): return (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) / np.sqrt(2)
def rel(x, y): return float(np.abs(np.asarray(x) - y).max() / max(np.abs(y).max(), 1e-300))
for shape in [(8, 4), (64, 16), (200, 16), (200, 40), (5000, 64)]:
    a = cg(*shape)
    q0, r0 = np.linalg.qr(a)
    res = P.householder_qr(a)
    print("hqr", shape, "R", rel(res.r, r0), "Q", rel(res.q, q0), "QR-A", rel(res.q @ res.r, a),
          "orth", np.abs(res.q.conj().T @ res.q - np.eye(shape[1])).max())
v, _ = np.linalg.qr(cg(150, 6)); a = cg(150, 4)
for ch in ["qr", "mlu", "polar"]:
    ref = O.two_stage(v, a, ch)
    res = P.two_stage_qr(v, a, choice=ch)
    print(ch, "q", rel(res.q, ref["q"]), "r", rel(res.r, ref["r"]), "s", rel(res.s, ref["s"]),
          "kt", res.diagnostics.kappa_t, ref["kappa_t"], "wn", res.diagnostics.wt_inv_norm, ref["wt_inv_norm"])
    print("   r diag", np.diag(res.r)[:4], np.diag(ref["r"])[:4])
