"""Section cycle counters of the fused chain factor inside two_stage_qr
(needs OTS_LIB=.../libots_timing.so, built by `make timing`)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 128
V = P.block_householder_qr([torch.randn((n, 64), dtype=torch.float64, device="cuda:0") for _ in range(k0 // 64)]).q.contiguous()
A = torch.randn((n, 64), dtype=torch.float64, device="cuda:0")
P.two_stage_qr(V, A); torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
NT.lib().ots_debug_counters(buf, 1)
ctx = NT.context(0); NT.lib().ots_set_profiling(ctx, 1)
P.two_stage_qr(V, A); torch.cuda.synchronize()
print(NT.profile(ctx))
NT.lib().ots_debug_counters(buf, 0)
tiles = buf[4]
print("tiles", tiles)
for i, nm in enumerate(["load", "sweep", "store", "tinv", "ntile", "pfact", "apply_nxt", "thread0_panel", "pf_load",
                        "pf_dlarfg", "pf_dots", "pf_update", "pf_store", "fused_x"]):
    print(f"{nm:13s} {buf[i] / max(tiles, 1):12.0f} cycles/tile")
