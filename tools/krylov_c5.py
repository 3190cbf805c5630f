"""BASELINE configs[4] block-Krylov sweep on one GPU: n = 2^24 (or argv[1]),
k = 64, A0 = N(0,1), 8 steps A <- L Q_prev (1D Laplacian, Dirichlet ends)
orthogonalised against the growing basis (k0 = 64 .. 512) on the
device-resident KrylovBasis, with and without the incremental Gram.  Device
time per step (CUDA events) and the final augmented loss / residual."""
import json, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_14449_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
k = 64
out = {}
for inc in (False, True):
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    A0 = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda")
    kb = P.KrylovBasis(n, 9 * k, device=0, incremental_gram=inc)
    kb.append(A0); del A0
    steps = []
    tot = 0.0
    for step in range(1, 9):
        qprev = kb.q[:, (step - 1) * k:step * k]
        Lq = 2.0 * qprev
        Lq[1:] -= qprev[:-1]
        Lq[:-1] -= qprev[1:]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = kb.append(Lq)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tot += ms
        steps.append(round(ms, 2))
        del Lq
    loss = P.orthonormality_defect(kb.q)
    out["incremental" if inc else "full_gram"] = {"step_ms": steps, "sweep_ms": round(tot, 1), "final_loss": loss}
    print(("incremental" if inc else "full_gram"), steps, "sweep", round(tot, 1), "ms, loss", loss, flush=True)
    del kb
    torch.cuda.empty_cache()
print(json.dumps(out))
