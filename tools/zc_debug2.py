import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2602_14449_b200 as P
from oracle import twostage_oracle as O
rng = np.random.default_rng(1)
def cg(n, m): return (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) / np.sqrt(2)
for k0 in [32, 40, 48]:
    v = np.linalg.qr(cg(3000, k0))[0]; a = cg(3000, 8)
    try:
        res = P.two_stage_qr(v, a); ref = O.two_stage(v, a, "qr")
        print("complex k0", k0, np.abs(res.q - ref["q"]).max())
    except Exception as e:
        print("complex k0", k0, "ERR", type(e).__name__, e)
for k0 in [80, 96]:
    v = np.linalg.qr(rng.standard_normal((3000, k0)))[0]; a = rng.standard_normal((3000, 8))
    res = P.two_stage_qr(v, a); ref = O.two_stage(v, a, "qr")
    print("real k0", k0, np.abs(res.q - ref["q"]).max())
# metrics with k=40 uses sym PW=64... real cholshift k=48
a = rng.standard_normal((3000, 48))
res = P.shifted_cholesky_qr(a); q0, r0 = O.cholqr_shifted(a)
print("real cholshift 48", np.abs(res.q - q0).max())
