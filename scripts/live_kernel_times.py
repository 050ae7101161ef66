"""Live per-kernel time of one config's fit (diagnostics): the fit runs as it does in bench.py
(graph replay, warm caches, real clocks) under torch.profiler (CUPTI kernel records), and the
kernel time per sweep is summed per kernel name, next to the wall time of the sweeps."""
import argparse
import collections
import json
import sys

import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
cfg = CONFIGS[args.config]
d = generate_torch(args.config, torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
Y, M, F = d["Y"], d["mask"], [f.clone() for f in d["init"]]
for _ in range(2):
    plan.fit(Y, M, cfg.alpha, cfg.beta, F, args.iters)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
plan.fit(Y, M, cfg.alpha, cfg.beta, F, args.iters)
e1.record()
torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / args.iters
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    plan.fit(Y, M, cfg.alpha, cfg.beta, F, args.iters)
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
first, last = None, None
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    name = ev.name.split("(")[0][:60]
    tot[name] += ev.device_time_total / 1e3
    cnt[name] += 1
    s, e = ev.time_range.start / 1e3, ev.time_range.end / 1e3
    first = s if first is None else min(first, s)
    last = e if last is None else max(last, e)
busy = sum(tot.values())
print(json.dumps({"config": args.config, "iters": args.iters, "ms_per_sweep_events": wall,
                  "ms_per_sweep_profiled_span": (last - first) / args.iters if first is not None else None,
                  "kernel_ms_per_sweep": busy / args.iters}))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print("%8.4f ms/sweep %6.1f launches/sweep %7.2f us/launch  %s" % (
        v / args.iters, cnt[k] / args.iters, 1e3 * v / cnt[k], k))
