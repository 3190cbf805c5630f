"""Per-entry parity of the row-sharded phases (simulated ranks on one GPU)
against the oracle: python tools/dist_probe.py WORLD N [K0 K]"""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import twostage_oracle as O  # noqa: E402
from paper_2602_14449_b200 import _device as D  # noqa: E402
from paper_2602_14449_b200 import _native as NT  # noqa: E402
from paper_2602_14449_b200 import workloads as W  # noqa: E402
from paper_2602_14449_b200.dist import LocalComm, NativePhases, run_phases  # noqa: E402

world, n = int(sys.argv[1]), int(sys.argv[2])
k0, k = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (128, 64)
rng = W.make_rng(5 + n + world)
v, _ = np.linalg.qr(W.normal_matrix(rng, n, k0))
a = W.normal_matrix(rng, n, k)
ref = O.two_stage(v, a, "qr", diagnostics=False)
splits = [0] + [n * (r + 1) // world for r in range(world)]
shared = LocalComm.make_shared(world)
outs = [None] * world


def run(rank):
    torch.cuda.set_device(0)
    r0, r1 = splits[rank], splits[rank + 1]
    V, A = D.to_device(v[r0:r1], 0), D.to_device(a[r0:r1], 0)
    Q, R, S = D.empty(r1 - r0, k, 0), D.zeros(k, k, 0), D.empty(k0, k, 0)
    ctx = NT.new_context(0)
    run_phases(NativePhases(0, ctx=ctx), LocalComm(rank, world, shared), r1 - r0, r0, k0, k, V, A, Q, R, S, "qr")
    torch.cuda.synchronize()
    outs[rank] = (Q.numpy(), R.numpy(), S.numpy(), NT.last_fast(ctx))


th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in th]
[t.join() for t in th]
q = np.vstack([o[0] for o in outs])
err = np.abs(q - ref["q"]) / (np.abs(ref["q"]) + 1e-4 * np.abs(ref["q"]).max())
i, j = np.unravel_index(np.argmax(err), err.shape)
rr = np.abs(outs[0][1] - ref["r"]) / (np.abs(ref["r"]) + 1e-4 * np.abs(ref["r"]).max())
print({"world": world, "n": n, "fast": [o[3] for o in outs], "q": float(err.max()), "at": (int(i), int(j)),
       "rows_over_3e-11": int((err.max(axis=1) > 3e-11).sum()), "r": float(rr.max()),
       "q_ref_entry": float(ref["q"][i, j]), "abs_err": float(abs(q[i, j] - ref["q"][i, j]))})
