import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2602_14449_b200 as P
from paper_2602_14449_b200 import workloads as W
from oracle import twostage_oracle as O
x = W.normal_matrix(W.make_rng(17), 20000, 80)
v = np.linalg.qr(W.normal_matrix(W.make_rng(18), 20000, 30))[0]
vd = torch.from_numpy(v).cuda(); ad = torch.from_numpy(x).cuda()
h = P.build_reflector(vd, "qr")
for cols in (16, 64, 80):
    ah = P.apply_reflector(h, ad[:, :cols].contiguous(), adjoint=True).cpu().numpy()
    bad = ~np.isfinite(ah)
    print(cols, "nonfinite", bad.sum(), "cols", np.unique(np.argwhere(bad)[:, 1])[:10], "rows", np.unique(np.argwhere(bad)[:, 0])[:5])
hn = P.build_reflector(v, "qr")
ahn = P.apply_reflector(hn, x, adjoint=True)
print("numpy path nonfinite", (~np.isfinite(ahn)).sum())
