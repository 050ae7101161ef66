"""Throughput of the App. B losses (N1) and of the split fit (N2) on a full-size configuration
(default c3: 1024 x 1024 x 384 CP, R = 32): per loss, ms per sweep of a fit, entries/s and the
streaming kernel's live fraction of the HBM roofline (algorithmic bytes: 4 B of Y + 1 B of mask
+ 4 B per entry of a per-entry parameter stream).  Data are drawn from each loss's own
likelihood around the config's planted mean.  python scripts/losses_bench.py [--config c3]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=5)
args = ap.parse_args()
cfg = CONFIGS[args.config]
dev = torch.device("cuda")
d = generate_torch(args.config, dev)
M = d["mask"]
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
peak = 6543.4
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except OSError:
    pass
g = torch.Generator(device=dev).manual_seed(11)
mean = torch.einsum(cfg.model, *d["truth"])
mean = mean / mean.mean() * 2.0
phi = torch.rand(mean.shape, generator=g, device=dev) * 3.5 + 0.5
ntr = torch.randint(1, 9, mean.shape, generator=g, device=dev).float()
lam = torch._standard_gamma(phi, generator=g) * (mean / phi)
data = {
    "negbin": torch.poisson(lam, generator=g),
    "bernoulli": (torch.rand(mean.shape, generator=g, device=dev) < mean / (1 + mean)).float(),
    "binomial": torch.binomial(ntr, mean / (1 + mean), generator=g),
    "js": torch.poisson(mean, generator=g),
}
cases = [("negbin", dict(param=2.0), None), ("negbin-phi_i", dict(), phi), ("bernoulli", {}, None),
         ("binomial", dict(param=8.0), None), ("binomial-n_i", dict(), ntr), ("js", {}, None)]


def run(name, fn, extra_bytes=0):
    fn(2)   # warm-up: >= 2 sweeps so that nef_fit's sweep graph is captured outside the timing
    torch.cuda.synchronize()
    nef.nef_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(args.iters)
    e1.record()
    torch.cuda.synchronize()
    kms, nl, byt = nef.nef_profile_read()
    nef.nef_profile_enable(False)
    ms = e0.elapsed_time(e1) / args.iters
    frac = (byt / nl) / (kms / nl / 1e3) / 1e9 / peak if nl else None
    print(json.dumps({"config": args.config, "case": name, "ms_per_sweep": ms,
                      "entries_per_s": cfg.n_entries / (ms / 1e3), "stream_kernel_ms_per_launch": kms / max(nl, 1),
                      "stream_roofline_frac": frac, "tc_lowerings": [L["tc"] for L in plan.describe()["lowerings"]]}))


for name, kw, aux in cases:
    kind = name.split("-")[0]
    Y = data[kind].contiguous()
    spec = nef.loss_spec(kind, aux=aux, **kw)
    F = [f.clone() for f in d["init"]]
    run(name + (" (per-entry parameter stream, +4 B/entry)" if aux is not None else ""),
        lambda k: plan.fit_ex(Y, M, spec, F, k, aux=aux))
# split fit (N2): train / validation / heldout labels from the config's mask
lab = torch.where(M != 0, torch.ones_like(M), torch.zeros_like(M))
u = torch.rand(M.shape, generator=g, device=dev)
lab = torch.where((lab == 1) & (u < 0.1), torch.full_like(M, 3), lab)
lab = torch.where((lab == 1) & (u >= 0.1) & (u < 0.145), torch.full_like(M, 2), lab)
Y = d["Y"]
spec = nef.loss_spec("ab", cfg.alpha, cfg.beta)
F = [f.clone() for f in d["init"]]
run("split fit (3 losses per sweep, P:497 rules off)",
    lambda k: plan.fit_split(Y, lab, spec, F, max_iters=k, min_rel_decrease=-1e300, val_patience=0))
