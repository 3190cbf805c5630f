"""seed_polar section counters (timing build), through build_reflector (Gram +
seed only: no factor / diag kernels contribute to the slots)."""
import ctypes as C, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n, k0 = 1 << 22, int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = torch.Generator(device="cuda"); g.manual_seed(21)
V = P.block_householder_qr([torch.randn((n, 64), generator=g, dtype=torch.float64, device="cuda")
                            for _ in range(k0 // 64)]).q.contiguous()
P.build_reflector(V, "polar"); torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
NT.lib().ots_debug_counters(buf, 1)
P.build_reflector(V, "polar"); torch.cuda.synchronize()
NT.lib().ots_debug_counters(buf, 0)
ms = lambda c: round(c / 1.965e6, 3)
print({"jacobi_ms": ms(buf[10]), "post_ms": ms(buf[11]), "newton_schulz_ms": ms(buf[12]), "lu_ms": ms(buf[13]),
       "sweeps": buf[15]})
