"""Throughput of the paper's own multi-index models at their data shapes (
synthetic Poisson data from Gamma factors, 10 % missing): one fit of K sweeps timed with CUDA
events, entries/s per full sweep and the fused kernel's fraction of the HBM roofline
(5 B/entry algorithmic).  python scripts/paper_models_bench.py [--steps 5]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle import nef_oracle as O  # noqa: E402  (factor shapes only)
from paper_2602_02759_b200 import nef  # noqa: E402

MODELS = [
    ("uber", "wr,dr,hr,irk,jrk->wdhij", (27, 7, 24, 400, 400), (10, 6), (1.0, 0.0)),
    ("icews", "ir,jr,ak,kr,tr->ijat", (249, 249, 20, 228), (25, 10), (1.0, 0.0)),
    ("wits", "er,ir,gr,tk,kr->eigt", (196, 196, 96, 29), (25, 10), (1.0, 0.0)),
]
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6650.0
dev = torch.device("cuda")
for name, ms, shape, ranks, (al, be) in MODELS:
    g = torch.Generator(device=dev).manual_seed(20260219)
    fs = O.factor_shapes(ms, shape, ranks)
    truth = [torch._standard_gamma(torch.full(s, 1.0, device=dev), generator=g) * 0.5 for s in fs]
    Y = torch.poisson(torch.einsum(ms, *truth), generator=g).float()
    M = (torch.rand(shape, generator=g, device=dev) >= 0.1).to(torch.uint8)
    F = [torch.rand(s, generator=g, device=dev) * 0.9 + 0.1 for s in fs]
    plan = nef.Plan(ms, shape, ranks)
    plan.fit(Y, M, al, be, F, 2)
    torch.cuda.synchronize()
    nef.nef_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.fit(Y, M, al, be, F, args.steps)
    e1.record()
    torch.cuda.synchronize()
    kms, kl, kb = nef.nef_profile_read()
    nef.nef_profile_enable(False)
    t = e0.elapsed_time(e1)
    n = Y.numel()
    gbs = (kb / kl) / (kms / kl / 1e3) / 1e9 if kl else None
    print(json.dumps({"model": name, "einsum": ms, "shape": shape, "ranks": ranks, "entries": n,
                      "sweeps": args.steps, "ms_per_sweep": t / args.steps,
                      "entries_per_s": n * args.steps / (t / 1e3),
                      "tc_lowerings": [L["tc"] for L in plan.describe()["lowerings"]],
                      "fused_launches": kl, "fused_GBps": gbs, "roofline_frac": gbs / peak if gbs else None}))
    del Y, M, F, truth, plan
    torch.cuda.empty_cache()
