import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
from bench import make_inputs
n, k0, k = 1 << 22, 128, 64
v, a = make_inputs(n, k0, k, 0)
z = torch.randn(k0, 32, dtype=torch.float64, device="cuda")
a[:, :32] = v @ z
a[:, 40:44] = a[:, 36:40]
for _ in range(3):
    res = P.two_stage_qr(v, a, choice="qr")
torch.cuda.synchronize()
ctx = NT.context(0); L = NT.lib()
L.ots_set_profiling(ctx, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ph = {}
for _ in range(5):
    res = P.two_stage_qr(v, a, choice="qr")
    for nm, ms in NT.profile(ctx):
        ph[nm] = ph.get(nm, 0.0) + ms / 5
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms": e0.elapsed_time(e1) / 5, "fast": NT.last_fast(ctx), "phases": {k_: round(v_, 3) for k_, v_ in ph.items()}}))
