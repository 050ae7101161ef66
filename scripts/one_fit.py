"""One nef_fit of a config (diagnostics, e.g. under ncu): python scripts/one_fit.py c5 2"""
import sys

import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[name]
d = generate_torch(name, torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
F = [f.clone() for f in d["init"]]
for _ in range(2):
    tr = plan.fit(d["Y"], d["mask"], cfg.alpha, cfg.beta, F, iters)
torch.cuda.synchronize()
print(name, list(tr))
