import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2602_14449_b200 as P
n, k0, k = 1 << 22, 64, 64
g = torch.Generator(device="cuda:0"); g.manual_seed(3)
d = 10.0 ** (4.0 * torch.rand(n, generator=g, dtype=torch.float64, device="cuda:0"))
V = torch.zeros((n, k0), dtype=torch.complex128, device="cuda:0")
V[:k0] = torch.diag(d[:k0].rsqrt()).to(torch.complex128)
A = torch.randn((n, k), generator=g, dtype=torch.complex128, device="cuda:0")
ip = P.InnerProduct.weighted(d)
u = P.initial_b_basis(ip, k0 + k)
for _ in range(2):
    P.b_two_stage_qr(V, A, u, ip)
torch.cuda.synchronize()
