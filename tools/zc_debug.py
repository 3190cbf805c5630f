import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O
rng = np.random.default_rng(1)
def cg(n, m): return (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) / np.sqrt(2)
for k in [8, 16, 24, 32, 33, 40, 48, 64]:
    for m in [500, 5000]:
        a = cg(m, k)
        try:
            res = P.shifted_cholesky_qr(a)
            q0, r0 = O.cholqr_shifted(a)
            print(k, m, "ok", np.abs(res.r - r0).max() / np.abs(r0).max(), np.abs(res.q - q0).max())
        except Exception as e:
            print(k, m, "ERR", type(e).__name__)
