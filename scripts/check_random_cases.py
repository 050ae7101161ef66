import sys; sys.path.insert(0, '.')
import numpy as np, torch
from tests.test_gpu_edges import _random_cases, _rel
from oracle import nef_oracle as O
from paper_2602_02759_b200 import nef
for pol in (0, 1):
    nef.nef_set_kernel_policy(pol)
    for c in _random_cases(200, 7):
        if c[1] not in [(143,76,108),(122,144,68),(74,140,140)]: continue
        ms, shape, ranks, ab, pm, seed = c
        rng = np.random.default_rng(seed)
        fs = O.factor_shapes(ms, shape, ranks)
        truth = [rng.gamma(1.0, 1.0, s) for s in fs]
        Y = (rng.poisson(O.contract(ms, truth)) + rng.gamma(2.0, 0.05, shape)).astype(np.float32)
        M = (rng.random(shape) >= pm).astype(np.uint8) if pm > 0 else None
        init = [rng.uniform(0.1, 1, s).astype(np.float32) for s in fs]
        plan = nef.Plan(ms, shape, ranks)
        F = [torch.from_numpy(f.copy()).cuda() for f in init]
        tr = plan.fit(torch.from_numpy(Y).cuda(), torch.from_numpy(M).cuda() if M is not None else None, ab[0], ab[1], F, 1)
        ref, rtr = O.fit(ms, Y, M, init, ab[0], ab[1], 1)
        print('policy', pol, shape, [round(_rel(f.cpu().numpy(), r) * 1e5, 2) for f, r in zip(F, ref)], 'x1e-5')
