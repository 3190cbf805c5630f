import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n = 1 << 20
g = torch.Generator(device="cuda:0"); g.manual_seed(1)
V = P.block_householder_qr([torch.randn((n, 64), generator=g, dtype=torch.float64, device="cuda:0") for _ in range(2)]).q.contiguous()
A = torch.randn((n, 64), generator=g, dtype=torch.float64, device="cuda:0")
for ch in ["qr", "mlu", "polar"]:
    P.two_stage_qr(V, A, choice=ch); torch.cuda.synchronize()
    buf = (C.c_ulonglong * 16)(); NT.lib().ots_debug_counters(buf, 1)
    P.two_stage_qr(V, A, choice=ch); torch.cuda.synchronize()
    NT.lib().ots_debug_counters(buf, 0)
    print(ch, "cta0", buf[10] / 1.96e6, "cta1", buf[11] / 1.96e6, "cta2: E", buf[12] / 1.96e6,
          "M", buf[13] / 1.96e6, "lmax", buf[14] / 1.96e6, "ms")
