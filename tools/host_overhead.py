import sys, time, cProfile, pstats, io
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n, k0, k = 1 << 20, 64, 32
g = torch.Generator(device="cuda:0"); g.manual_seed(1)
V = torch.linalg.qr(torch.randn((n, k0), generator=g, dtype=torch.float64, device="cuda:0"))[0].contiguous()
A = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda:0")
for _ in range(3): P.two_stage_qr(V, A)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter(); P.two_stage_qr(V, A); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("wall ms median", sorted(ts)[10] * 1e3)
ctx = NT.context(0)
NT.lib().ots_set_profiling(ctx, 1)
P.two_stage_qr(V, A); torch.cuda.synchronize()
prof = dict(NT.profile(ctx)); print("gpu phases sum", sum(prof.values()))
NT.lib().ots_set_profiling(ctx, 0)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): P.two_stage_qr(V, A)
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(18); print(s.getvalue()[:3500])
