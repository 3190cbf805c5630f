"""One-off: per-entry parity of the headline call (n = 2^24, k0 = 128, k = 64)
against the CPU oracle on the same inputs (needs ~80 GB of host RAM and a few
minutes of host LAPACK).  V is an orthonormal basis produced on the GPU and
handed to both sides as the same float64 array."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_14449_b200 as P  # noqa: E402
from oracle import twostage_oracle as O  # noqa: E402
from paper_2602_14449_b200 import _native as NT  # noqa: E402
from bench import make_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
k0, k = 128, 64
V, A = make_inputs(n, k0, k, 0)
res = P.two_stage_qr(V, A)
fast = NT.last_fast(NT.context(0))
q, r, s = res.q.cpu().numpy(), res.r.cpu().numpy(), res.s.cpu().numpy()
v, a = V.cpu().numpy(), A.cpu().numpy()
del V, A, res
torch.cuda.empty_cache()
t0 = time.time()
ref = O.two_stage(v, a, "qr", diagnostics=False)
t_cpu = time.time() - t0


def rel(x, y, floor=1e-4):
    scale = float(np.abs(y).max())
    out = 0.0
    for i in range(0, x.shape[0], 1 << 20):          # blockwise: no n x k temporaries beyond 1M rows
        xs, ys = x[i:i + (1 << 20)], y[i:i + (1 << 20)]
        out = max(out, float((np.abs(xs - ys) / (np.abs(ys) + floor * scale)).max()))
    return out


print(json.dumps({"n": n, "k0": k0, "k": k, "direct_q": fast, "q": rel(q, ref["q"]), "r": rel(r, ref["r"]),
                  "s": rel(s, ref["s"]), "oracle_seconds": round(t_cpu, 1)}))
