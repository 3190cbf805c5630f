"""One two_stage_qr call at a chosen size on HBM-resident inputs (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_14449_b200 as P  # noqa: E402
from paper_2602_14449_b200 import _native as NT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--k0", type=int, default=128)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--choice", default="qr")
ap.add_argument("--vgen", default="ots", help="ots | torch (cuSOLVER QR) | eye ([I; 0]) | rot ([W; 0], W random orthogonal)")
a = ap.parse_args()
g = torch.Generator(device="cuda:0")
g.manual_seed(1)
G = torch.randn((a.n, a.k0), generator=g, dtype=torch.float64, device="cuda:0")
if a.vgen == "rot":      # [W; 0] with W a random orthogonal k0 x k0: a non-trivial seed
    V = torch.zeros((a.n, a.k0), dtype=torch.float64, device="cuda:0")
    V[:a.k0].copy_(torch.linalg.qr(torch.randn((a.k0, a.k0), generator=g, dtype=torch.float64,
                                               device="cuda:0"))[0])
elif a.vgen == "eye":      # exactly orthonormal [I; 0] (no setup kernels)
    V = torch.zeros((a.n, a.k0), dtype=torch.float64, device="cuda:0")
    V[:a.k0].copy_(torch.eye(a.k0, dtype=torch.float64))
elif a.vgen == "torch":
    V = torch.linalg.qr(G)[0].contiguous()
else:
    V = P.block_householder_qr([G[:, i:i + 64].contiguous() for i in range(0, a.k0, 64)]).q.contiguous()
A = torch.randn((a.n, a.k), generator=g, dtype=torch.float64, device="cuda:0")
ctx = NT.context(0)
NT.lib().ots_set_profiling(ctx, 1)
for _ in range(a.reps):
    r = P.two_stage_qr(V, A, choice=a.choice)
    torch.cuda.synchronize()
    print({k: round(v, 3) for k, v in NT.profile(ctx)}, flush=True)
