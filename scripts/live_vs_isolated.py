"""Why the streaming kernel is slower inside a fit than under ncu: time the
c5 factor updates (a) back to back inside a 10-sweep fit (live CUDA events, nef_profile) and (b)
one at a time after 2 s of idle GPU (the way ncu's serialised replays see them), with the SM clock
sampled by nvidia-smi during each.  python scripts/live_vs_isolated.py"""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402


def smi():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
        return out.strip()
    except Exception:
        return None


cfg = CONFIGS["c5"]
d = generate_torch("c5", torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
Y, M = d["Y"], d["mask"]
F = [f.clone() for f in d["init"]]
plan.fit(Y, M, cfg.alpha, cfg.beta, F, 3)
torch.cuda.synchronize()
nef.nef_profile_enable(True)
plan.fit(Y, M, cfg.alpha, cfg.beta, F, 10)
s_live = smi()
torch.cuda.synchronize()
kms, nl, _ = nef.nef_profile_read()
nef.nef_profile_enable(False)
print(json.dumps({"what": "live, 10-sweep fit (sentinel stream, all passes)", "ms_per_launch": kms / nl,
                  "launches": nl, "smi_at_end": s_live}))
for ell in range(3):
    for rep in range(2):
        time.sleep(2.0)
        G = [f.clone() for f in F]
        torch.cuda.synchronize()
        nef.nef_profile_enable(True)
        plan.update(ell, Y, None, cfg.alpha, cfg.beta, G)   # unmasked: the MM = 0 kernel the fit streams
        torch.cuda.synchronize()
        kms, nl, _ = nef.nef_profile_read()
        nef.nef_profile_enable(False)
        print(json.dumps({"what": "isolated update ell=%d after 2 s idle (raw Y, MM = 0)" % ell, "ms": kms / max(nl, 1),
                          "smi_after": smi()}))
    nef.nef_profile_enable(True)
    G = [f.clone() for f in F]
    for rep in range(6):
        plan.update(ell, Y, None, cfg.alpha, cfg.beta, G)
    torch.cuda.synchronize()
    kms, nl, _ = nef.nef_profile_read()
    nef.nef_profile_enable(False)
    print(json.dumps({"what": "update ell=%d x6 back to back" % ell, "ms": kms / max(nl, 1), "smi_after": smi()}))
