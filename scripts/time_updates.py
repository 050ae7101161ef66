"""Time each factor update (one streaming launch + small kernels) of a config, per kernel policy."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--policies", default="0,1")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--nomask", action="store_true")
args = ap.parse_args()
cfg = CONFIGS[args.config]
d = generate_torch(args.config, torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
desc = plan.describe()
Y, M, F = d["Y"], (None if args.nomask else d["mask"]), d["init"]
res = {}
for pol in [int(p) for p in args.policies.split(",")]:
    nef.nef_set_kernel_policy(pol)
    for ell in range(len(F)):
        G = [f.clone() for f in F]
        plan.update(ell, Y, M, cfg.alpha, cfg.beta, G)   # warm
        torch.cuda.synchronize()
        nef.nef_profile_enable(True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            plan.update(ell, Y, M, cfg.alpha, cfg.beta, G)
        e1.record()
        torch.cuda.synchronize()
        kms, kl, kb = nef.nef_profile_read()
        nef.nef_profile_enable(False)
        t = e0.elapsed_time(e1) / args.reps
        L = desc["lowerings"][ell]
        res["pol%d_ell%d" % (pol, ell)] = dict(rows=L["row_idx"], tc=L["tc"], layout=L["tc_layout"], ms_update=t,
                                               ms_kernel=kms / kl, GBps=kb / kl / (kms / kl / 1e3) / 1e9)
        print(json.dumps({"policy": pol, "ell": ell, **res["pol%d_ell%d" % (pol, ell)]}), flush=True)
