"""Small-call latency probe (C1 shape by default): wall and device time per
two_stage_qr on resident CUDA tensors, per-phase device times, launches."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n, k0, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (100000, 32, 16)))
g = torch.Generator(device="cuda:0"); g.manual_seed(1)
V = P.householder_qr(torch.randn((n, k0), generator=g, dtype=torch.float64, device="cuda:0")).q.contiguous()
A = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda:0")
for _ in range(5): P.two_stage_qr(V, A)
torch.cuda.synchronize()
ts, ds = [], []
for _ in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(); P.two_stage_qr(V, A); e1.record(); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0); ds.append(e0.elapsed_time(e1))
ts.sort(); ds.sort()
print(f"n={n} k0={k0} k={k}: wall {ts[15]*1e3:.3f} ms, events {ds[15]:.3f} ms")
ctx = NT.context(0)
print("launches", NT.lib().ots_last_launch_count(ctx))
NT.lib().ots_set_profiling(ctx, 1)
P.two_stage_qr(V, A); torch.cuda.synchronize()
print([(a, round(b, 4)) for a, b in NT.profile(ctx)])
NT.lib().ots_set_profiling(ctx, 0)
