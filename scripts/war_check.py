"""Diagnostics: run each c5 factor update with the buffer WAR wait on (default) and off
(NEF_TC_DBG=8 set by the caller) and print a checksum of the resulting factor bits, so two
runs can be compared for bit-identity."""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = CONFIGS[name]
d = generate_torch(name, torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
for rep in range(3):
    F = [f.clone() for f in d["init"]]
    tr = plan.fit(d["Y"], d["mask"], cfg.alpha, cfg.beta, F, 2)
    torch.cuda.synchronize()
    h = hashlib.sha256(b"".join(f.cpu().numpy().tobytes() for f in F)).hexdigest()[:16]
    print(name, "rep", rep, "factors sha", h, "trace", list(tr))
