"""Throughput of batched random restarts (N4): S fits of one full-size config sharing each
streamed pass (nef_fit_restarts), S = 1..4.  Prints one JSON line per S: ms per sweep (all
restarts), restart-sweeps of entries per second, and the streaming kernel's live CUDA-event time
per launch (one launch carries all S restarts).
    python scripts/restarts_bench.py --config c5 --iters 5"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--max-restarts", type=int, default=4)
args = ap.parse_args()
cfg = CONFIGS[args.config]
dev = torch.device("cuda")
d = generate_torch(args.config, dev)
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
spec = nef.loss_spec("ab", cfg.alpha, cfg.beta)
g = torch.Generator(device=dev).manual_seed(5)
for S in range(1, args.max_restarts + 1):
    Fs = [[f.clone() if r == 0 else torch.rand(f.shape, generator=g, device=dev) * 0.9 + 0.1 for f in d["init"]]
          for r in range(S)]
    ws = torch.empty(nef.nef_restarts_workspace_bytes(plan.h, S), dtype=torch.uint8, device=dev)
    nef.nef_fit_restarts(plan.h, d["Y"], d["mask"], spec, 1e-12, Fs, 1, ws)   # warm-up
    torch.cuda.synchronize()
    nef.nef_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tr = nef.nef_fit_restarts(plan.h, d["Y"], d["mask"], spec, 1e-12, Fs, args.iters, ws)
    e1.record()
    torch.cuda.synchronize()
    kms, nl, _ = nef.nef_profile_read()
    nef.nef_profile_enable(False)
    ms = e0.elapsed_time(e1) / args.iters
    print(json.dumps({"config": args.config, "restarts": S, "ms_per_sweep": ms,
                      "restart_entries_per_s": S * cfg.n_entries / (ms / 1e3),
                      "stream_kernel_ms_per_launch": kms / max(nl, 1), "launches": nl,
                      "final_losses": [float(x) for x in tr[:, -1]]}))
    del ws, Fs
    torch.cuda.empty_cache()
