"""Section cycle counters of the Gram-form level-0 factor (gsweep.inc) inside
two_stage_qr (needs OTS_LIB=.../libots_timing.so, built by `make timing`)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
from bench import make_inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
V, A = make_inputs(n, 128, 64, 0)
P.two_stage_qr(V, A); torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
NT.lib().ots_debug_counters(buf, 1)
ctx = NT.context(0); NT.lib().ots_set_profiling(ctx, 1)
P.two_stage_qr(V, A); torch.cuda.synchronize()
print(NT.profile(ctx))
NT.lib().ots_debug_counters(buf, 0)
tiles = buf[4]
print("tiles", tiles)
for i, nm in enumerate(["gram", "sweep", "inverses", "rho+out", "ntile", "S1 (64/tile)"]):
    print(f"{nm:13s} {buf[i] / max(tiles, 1):12.0f} cycles/tile")
