"""Diagnostics: worst relative factor error after one sweep vs the float64 oracle on the TF32
path, across bond sizes / models / (alpha, beta)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import nef_oracle as O
from paper_2602_02759_b200 import nef


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30)))


nef.nef_set_kernel_policy(0)
for ms, shape, ranks_list in [("ia,jb,kc,abc->ijk", (128, 128, 128), [(8, 8, 8), (12, 12, 12), (14, 14, 14), (16, 16, 16)]),
                              ("ir,jr,kr->ijk", (128, 128, 128), [(8,), (12,), (14,), (16,), (32,)])]:
    for ranks in ranks_list:
        for ab in [(1.0, 1.0), (1.0, 0.0)]:
            rng = np.random.default_rng(5)
            fs = O.factor_shapes(ms, shape, ranks)
            truth = [rng.gamma(1.0, 1.0, s) for s in fs]
            Y = (rng.poisson(O.contract(ms, truth)) + rng.gamma(2.0, 0.05, shape)).astype(np.float32)
            init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
            plan = nef.Plan(ms, shape, ranks)
            F = [torch.from_numpy(f.copy()).cuda() for f in init]
            plan.fit(torch.from_numpy(Y).cuda(), None, ab[0], ab[1], F, 1)
            ref, _ = O.fit(ms, Y, None, init, ab[0], ab[1], 1)
            tc = [L["tc"] for L in plan.describe()["lowerings"]]
            print(ms[:10], ranks, ab, tc, [round(rel(f.cpu().numpy(), r) * 1e5, 2) for f, r in zip(F, ref)], "x1e-5", flush=True)
