"""Seed timing for the polar choice at the C3 shape (n=2^22, k0=128, k=64)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n, k0, k = 1 << 22, 128, 64
g = torch.Generator(device="cuda"); g.manual_seed(21)
V = P.block_householder_qr([torch.randn((n, 64), generator=g, dtype=torch.float64, device="cuda") for _ in range(2)]).q.contiguous()
A = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda")
ctx = NT.context(0)
for ch in ("qr", "polar"):
    P.two_stage_qr(V, A, choice=ch)
    NT.lib().ots_set_profiling(ctx, 1)
    P.two_stage_qr(V, A, choice=ch); torch.cuda.synchronize()
    prof = NT.profile(ctx)
    print(ch, round(sum(b for _, b in prof), 2), [(a, round(b, 2)) for a, b in prof])
    NT.lib().ots_set_profiling(ctx, 0)
