"""Per-mode timing of one config (diagnostics): factor updates (streaming pass without loss),
loss-only pass, one full fit sweep (first pass carries the loss), fused-kernel time via the
library's live CUDA-event profile."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = CONFIGS[args.config]
d = generate_torch(args.config, torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
Y, M, F = d["Y"], d["mask"], [f.clone() for f in d["init"]]


def timed(fn, label):
    fn()
    torch.cuda.synchronize()
    nef.nef_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    kms, kl, kb = nef.nef_profile_read()
    nef.nef_profile_enable(False)
    print(json.dumps({"config": args.config, "what": label, "ms": e0.elapsed_time(e1) / args.reps,
                      "fused_ms_per_launch": kms / max(kl, 1), "fused_launches_per_call": kl / args.reps,
                      "GBps": (kb / kl) / (kms / kl / 1e3) / 1e9 if kl else None}), flush=True)


for ell in range(len(F)):
    timed(lambda: plan.update(ell, Y, M, cfg.alpha, cfg.beta, F), "update ell=%d" % ell)
timed(lambda: plan.loss(Y, M, cfg.alpha, cfg.beta, F), "loss only")
timed(lambda: plan.fit(Y, M, cfg.alpha, cfg.beta, F, 1), "fit iters=1")
timed(lambda: plan.fit(Y, M, cfg.alpha, cfg.beta, F, 4), "fit iters=4")
