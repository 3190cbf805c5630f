"""Phase times of one complex128 two_stage_qr call (configs[3] shape) on HBM-resident inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
k0 = k = 64
g = torch.Generator(device="cuda:0"); g.manual_seed(1)
G = torch.randn((n, k0), generator=g, dtype=torch.complex128, device="cuda:0")
V = (torch.linalg.qr(G)[0] if os.environ.get('PROF_TORCHV') else P.householder_qr(G).q).contiguous()
A = torch.randn((n, k), generator=g, dtype=torch.complex128, device="cuda:0")
ctx = NT.context(0)
NT.lib().ots_set_profiling(ctx, 1)
for _ in range(2):
    try:
        P.two_stage_qr(V, A)
    except Exception as exc:   # timing-only experiment libraries may break the checks
        print('call failed:', type(exc).__name__)
    torch.cuda.synchronize()
    print({kk: round(v, 3) for kk, v in NT.profile(ctx)}, flush=True)
