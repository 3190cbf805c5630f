"""Section cycle counters of the Gram-form level-0 factor (gsweep.inc) inside
two_stage_qr (needs OTS_LIB=.../libots_timing.so, built by `make timing`)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
from bench import make_inputs
os.environ.setdefault("OTS_GSWEEP", "1")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
if os.environ.get("GS_CPU_V"):   # probe libraries compute wrong results: orthonormalise on the host
    import numpy as np
    rng = np.random.default_rng(5)
    V = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, 128)))[0]).cuda()
    A = torch.from_numpy(rng.standard_normal((n, 64))).cuda()
else:
    V, A = make_inputs(n, 128, 64, 0)
try:
    P.two_stage_qr(V, A)
except Exception as exc:
    print('warm-up:', exc)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
NT.lib().ots_debug_counters(buf, 1)
ctx = NT.context(0); NT.lib().ots_set_profiling(ctx, 1)
try:
    P.two_stage_qr(V, A)
except Exception as exc:
    print('call:', exc)
torch.cuda.synchronize()
print(NT.profile(ctx))
NT.lib().ots_debug_counters(buf, 0)
tiles = buf[4]
print("tiles", tiles)
for i, nm in enumerate(["gram", "sweep", "rho+out", "-", "ntile", "phaseA(w0)", "B window", "C window(7)", "B w1", "Bp w3", "Tpp w5", "w0 in B"]):
    print(f"{nm:13s} {buf[i] / max(tiles, 1):12.0f} cycles/tile")
ev = (C.c_longlong * 64)()
try:
    NT.lib().ots_gs_event_log(ev)
    names = ["A start(w0)", "A end(w0)", "B1 out w0", "B1 out w1", "B2 out w0", "B2 out w1"]
    for p in range(8):
        row = [ev[p * 8 + k] for k in range(6)]
        base = row[0]
        print(f"panel {p}: " + " ".join(f"{nm}={v - base}" for nm, v in zip(names, row)))
except AttributeError:
    pass
