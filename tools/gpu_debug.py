"""Quick GPU smoke of the CUDA path vs the oracle (debug helper)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O
from paper_2602_14449_b200 import workloads as W

def rel(x, y):
    return float(np.abs(np.asarray(x) - np.asarray(y)).max() / max(np.abs(y).max(), 1e-300))

for (n, k0, k) in [(64, 8, 8), (500, 16, 8), (5000, 32, 16), (20000, 64, 32), (70000, 128, 64)]:
    rng = W.make_rng(7 + n)
    v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
    a = W.normal_matrix(rng, n, k)
    # intra QR alone
    try:
        q = P.householder_qr(a)
        qr_ref = O.lapack_qr(a)
        print(f"hqr n={n} k={k}: dq={rel(q.q, qr_ref[0]):.2e} dr={rel(q.r, qr_ref[1]):.2e}", flush=True)
    except Exception as e:
        print("hqr fail", type(e).__name__, e, flush=True)
    for ch in ("qr", "mlu", "polar"):
        try:
            t0 = time.time()
            res = P.two_stage_qr(v, a, choice=ch)
            t1 = time.time()
            ref = O.two_stage(v, a, ch)
            print(f"n={n} k0={k0} k={k} {ch}: dq={rel(res.q, ref['q']):.2e} dr={rel(res.r, ref['r']):.2e} "
                  f"ds={rel(res.s, ref['s']):.2e} kt={res.diagnostics.kappa_t:.6f}/{ref['kappa_t']:.6f} "
                  f"wn={res.diagnostics.wt_inv_norm:.6f}/{ref['wt_inv_norm']:.6f} t={t1-t0:.3f}s", flush=True)
        except Exception as e:
            import traceback; traceback.print_exc()
            print("FAIL", n, k0, k, ch, type(e).__name__, e, flush=True)
