import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2602_14449_b200 as P
from paper_2602_14449_b200.core import gram, update
g2 = np.load('tests/golden/golden_r02.npz')
v, a = g2['reorth_c/v'], g2['reorth_c/a']
s = gram(v, a).cpu().numpy(); print('s', np.abs(s - v.conj().T @ a).max())
ga = gram(a).cpu().numpy(); print('gram(a)', np.abs(ga - a.conj().T @ a).max())
z = (np.random.randn(6, 6) + 1j * np.random.randn(6, 6))
x = update(a, z).cpu().numpy(); print('update B=None', np.abs(x - a @ z).max())
zt = torch.from_numpy(z).cuda().mH
x = update(a, zt).cpu().numpy(); print('update mH', np.abs(x - a @ z.conj().T).max())
x = update(v, -s, a).cpu().numpy(); print('update B', np.abs(x - (a - v @ s)).max())
res = P.cholqr_two_stage(v, a)
print('q', np.abs(res.q - g2['cholqr_c/q']).max(), 'r', np.abs(res.r - g2['cholqr_c/r']).max(), 's', np.abs(res.s - g2['cholqr_c/s']).max())
