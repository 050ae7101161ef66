import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import nef_oracle as O
from tests.test_gpu_edges import _random_cases
def rn(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return (((b + 0x1000) & 0xFFFFE000).astype(np.uint32)).view(np.float32).astype(np.float64)
def strat(x, axis_len):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    j = (np.arange(b.shape[-1]) % 16).astype(np.uint64)
    d = 0x100 + 0x200 * j
    return (((b + d) & 0xFFFFE000).astype(np.uint32)).view(np.float32).astype(np.float64)
c = [c for c in _random_cases(200, 11) if c[1] == (87, 64, 76)][0]
ms, shape, ranks, ab, pm, seed = c
rng = np.random.default_rng(seed)
fs = O.factor_shapes(ms, shape, ranks)
truth = [rng.gamma(1.0, 1.0, s) for s in fs]
Y = (rng.poisson(O.contract(ms, truth)) + rng.gamma(2.0, 0.05, shape)).astype(np.float32)
M = (rng.random(shape) >= pm).astype(np.uint8)
init = [rng.uniform(0.1, 1, s).astype(np.float64) for s in fs]
# update sequence: factors 0,1 first (use oracle values), then factor 2 (kc): rows k, bond (a,b), cols (i,j)
th = [f.copy() for f in init]
for ell in range(2):
    th[ell] = O.update_factor(ms, Y, M, th, ell, *ab)
A, B, C, G = th
U = np.einsum('kc,abc->kab', C, G).reshape(shape[2], -1)          # k x (a,b)
V = np.einsum('ia,jb->ijab', A, B).reshape(shape[0]*shape[1], -1)  # (i,j) x (a,b)
X = Y.transpose(2,0,1).reshape(shape[2], -1).astype(np.float64)
Mk = M.transpose(2,0,1).reshape(shape[2], -1).astype(np.float64)
S = U @ V.T
N = (Mk * X) @ V; D = (Mk * S) @ V
Vr = rn(V.astype(np.float32)); Se = U @ Vr.T
Pa = Mk * strat(X, 16); Pb = Mk * rn(Se)
Ne = Pa @ Vr; De = Pb @ Vr
print('N rel', np.max(np.abs(Ne-N)/np.abs(N)), 'D rel', np.max(np.abs(De-D)/np.abs(D)))
# the Q -> factor epilogue: Num[k,c] = sum_ab Q[k,ab] G[a,b,c]; ratio
Gm = G.reshape(-1, G.shape[2])
num = N @ Gm; den = D @ Gm; nume = Ne @ Gm; dene = De @ Gm
print('factor ratio rel err', np.max(np.abs(nume/dene - num/den)/(num/den)))
print('X range', X.min(), X.max(), 'S row cv', np.mean(np.std(S,1)/np.mean(S,1)))
for name, Pa_, V_ in [("strat Pa, exact V", Mk*strat(X,16), V), ("exact Pa, RN V", Mk*X, Vr), ("RN Pa, exact V", Mk*rn(X), V)]:
    Ne2 = Pa_ @ V_
    print(name, 'N rel', np.max(np.abs(Ne2-N)/np.abs(N)))
print('V per-column cv', np.std(V,0)/np.mean(V,0))
print('rows of N with worst err', np.argsort(-np.max(np.abs(Ne-N)/np.abs(N),1))[:5], 'min |N|', np.min(np.abs(N)), 'median', np.median(np.abs(N)))
