"""Factor-update timing of CP shapes with the same entry count and different row strides
(diagnostics for the layout-1 TMA pattern): python scripts/shape_sweep.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

cfg = CONFIGS["c5"]
for shape in [(2048, 2048, 1024), (4096, 1024, 1024), (8192, 512, 1024), (2048, 1024, 2048), (1024, 4096, 1024)]:
    d = generate_torch("c5", torch.device("cuda"), shape=shape)
    plan = nef.Plan(cfg.model, shape, cfg.ranks)
    F = [f.clone() for f in d["init"]]
    for ell in range(3):
        plan.update(ell, d["Y"], d["mask"], cfg.alpha, cfg.beta, F)
        torch.cuda.synchronize()
        nef.nef_profile_enable(True)
        for _ in range(3):
            plan.update(ell, d["Y"], d["mask"], cfg.alpha, cfg.beta, F)
        torch.cuda.synchronize()
        kms, kl, kb = nef.nef_profile_read()
        nef.nef_profile_enable(False)
        L = plan.describe()["lowerings"][ell]
        print(json.dumps({"shape": shape, "ell": ell, "layout": L["tc_layout"], "ms": kms / kl,
                          "GBps_5B": kb / kl / (kms / kl / 1e3) / 1e9}), flush=True)
    del d, plan, F
    torch.cuda.empty_cache()
