"""Phase profile of one two_stage_qr at (n, k0, k) with V from the block QR
and, optionally, a supplied Gram (incremental path)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import _native as NT
n, k0, k = (int(x) for x in sys.argv[1:4])
g = torch.Generator(device="cuda"); g.manual_seed(3)
kb = P.KrylovBasis(n, k0 + k, device=0, incremental_gram=True)
for c in range(0, k0, 64):
    kb.append(torch.randn((n, 64), generator=g, dtype=torch.float64, device="cuda"))
A = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda")
V = kb.q
ctx = NT.context(0)
for mode in ("full", "gram"):
    for rep in range(2):
        NT.lib().ots_set_profiling(ctx, 1 if rep else 0)
        if mode == "full":
            P.two_stage_qr(V, A)
        else:
            kb2 = kb  # supplied Gram
            from paper_2602_14449_b200.twostage import _run_two_stage
            from paper_2602_14449_b200 import _device as D
            Vd = D.DMat(kb.buf, k0, ld=kb.ldb); Ad = D.to_device(A, 0)
            Q, R, S = D.empty(n, k, 0), D.zeros(k, k, 0), D.empty(k0, k, 0)
            _run_two_stage(0, Vd, Ad, Q, R, S, "qr", "householder", None, False, gram=kb.G[:k0, :k0])
        torch.cuda.synchronize()
    prof = NT.profile(ctx)
    print(mode, round(sum(b for _, b in prof), 2), [(a, round(b, 2)) for a, b in prof])
NT.lib().ots_set_profiling(ctx, 0)
