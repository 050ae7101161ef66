import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import nef_oracle as O
def rn(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return b.view(np.float32).astype(np.float64)
ms, shape, ranks = "ia,jb,kc,abc->ijk", (128,128,128), (12,12,12)
rng = np.random.default_rng(5)
fs = O.factor_shapes(ms, shape, ranks)
truth = [rng.gamma(1.0, 1.0, s) for s in fs]
Y = (rng.poisson(O.contract(ms, truth)) + rng.gamma(2.0, 0.05, shape)).astype(np.float32)
init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
A, B, C, G = [f.astype(np.float64) for f in init]
V = np.einsum('jb,kc,abc->jka', B, C, G).reshape(-1, 12)     # (j,k) x a
V32 = V.astype(np.float32).astype(np.float64)
X = Y.reshape(128, -1).astype(np.float64)
U = A
S = U @ V.T
N = X @ V; D = S @ V
ex = A * N / D
for name, Vs, Vn in [("RN V everywhere", rn(V32), rn(V32)), ("exact V in S, RN V in N/D", V32, rn(V32)), ("RN V in S only", rn(V32), V32)]:
    Se = U @ Vs.T
    Pa = rn(X); Pb = rn(Se)
    Ne = Pa @ Vn; De = Pb @ Vn
    up = A * Ne / De
    print(name, np.max(np.abs(up - ex) / ex))
