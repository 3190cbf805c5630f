"""Phase profile of one complex128 two_stage_qr at the C4 shape."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n, k0, k = 1 << 22, 64, 64
g = torch.Generator(device="cuda"); g.manual_seed(41)
G = torch.complex(torch.randn((n, k0), generator=g, dtype=torch.float64, device="cuda"),
                  torch.randn((n, k0), generator=g, dtype=torch.float64, device="cuda"))
V = torch.linalg.qr(G)[0].contiguous(); del G   # tool input only
A = torch.complex(torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda"),
                  torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda"))
ctx = NT.context(0)
P.two_stage_qr(V, A)
NT.lib().ots_set_profiling(ctx, 1)
P.two_stage_qr(V, A); torch.cuda.synchronize()
prof = NT.profile(ctx)
print(round(sum(b for _, b in prof), 2), [(a, round(b, 2)) for a, b in prof])
