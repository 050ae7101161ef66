"""Print the tcgen05 kernel's per-tile pipeline timeline (CTA (0,0)) for one factor update.
Needs the -DNEF_TRACE=1 build: scripts/build_variants.sh trace="-DNEF_TRACE=1", then run with
NEF_LIB=paper_2602_02759_b200/libnef_trace.so (or copy it over libnef.so)."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from nef_inputs import CONFIGS, generate_torch  # noqa: E402
from paper_2602_02759_b200 import nef  # noqa: E402

EV = ["TMA", "VG_START", "VG_DONE", "MMA1", "MMA23", "EW_S", "EW_Y", "EW_PEMPTY", "EW_DONE", "VG_ISSUED", "EW_LDW",
      "EW_MATH"]
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--ell", type=int, default=0)
ap.add_argument("--first", type=int, default=200)
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--nomask", action="store_true", help="unmasked update (the MM = 0 kernel the fit runs on the sentinel copy)")
args = ap.parse_args()
cfg = CONFIGS[args.config]
d = generate_torch(args.config, torch.device("cuda"))
plan = nef.Plan(cfg.model, cfg.shape, cfg.ranks)
F = [f.clone() for f in d["init"]]
M = None if args.nomask else d["mask"]
plan.update(args.ell, d["Y"], M, cfg.alpha, cfg.beta, F)
tr = torch.zeros(1024 * 32, dtype=torch.int64, device="cuda")
nef.nef_debug_trace(tr)
plan.update(args.ell, d["Y"], M, cfg.alpha, cfg.beta, F)
torch.cuda.synchronize()
nef.nef_debug_trace(None)
full = tr.cpu().numpy().reshape(1024, 32).astype(np.int64)
t = full[:, :len(EV)]
valid = (t[:1023, EV.index("EW_DONE")] > 0).sum()   # (row 1023 holds the launch phases)
print("tiles traced", valid)
ph = full[1023, :13]
if ph[0] > 0:
    print("direct-V loader lane (cycles after entry): starts %d, run cursor initialised %d, first table row known %d, "
          "first TMA issued %d" % (ph[10] - ph[0], ph[11] - ph[0], ph[12] - ph[0], ph[5] - ph[0]))
    print("prologue (cycles after entry): first V TMA issued %d, constant rows issued %d landed %d, "
          "EW warp 0 U stored %d, issuer saw U %d, first raw V landed (VG_START) %d"
          % (ph[5] - ph[0], ph[9] - ph[0], ph[6] - ph[0], ph[7] - ph[0], ph[8] - ph[0], t[0, EV.index("VG_START")] - ph[0]))
if ph[0] > 0:   # launch phases of CTA (0, 0), cycles after kernel entry
    last = t[valid - 1, EV.index("EW_DONE")] if valid > 0 else ph[0]
    print("launch phases (cycles after entry): setup done %d, first TMA %d, first MMA1 %d, first EW_DONE %d, "
          "last EW_DONE %d, last N/D retired %d, partials written %d, all roles done %d"
          % (ph[1] - ph[0], t[0, EV.index("TMA")] - ph[0], t[0, EV.index("MMA1")] - ph[0],
             t[0, EV.index("EW_DONE")] - ph[0], last - ph[0], ph[2] - ph[0], ph[3] - ph[0], ph[4] - ph[0]))
lo, hi = min(args.first, max(valid - 2, 0)), min(args.first + args.n, valid - 1)
base = t[lo, EV.index("MMA1")]
print("tile " + " ".join("%9s" % e for e in EV))
for i in range(lo, hi):
    print("%4d " % i + " ".join("%9d" % (t[i, j] - base) for j in range(len(EV))))
per = np.diff(t[lo:hi + 1, EV.index("EW_DONE")])
print("cycles per tile (EW_DONE to EW_DONE): median %d" % np.median(per))
for a_, b_ in [("MMA1", "EW_S"), ("EW_S", "EW_Y"), ("EW_Y", "EW_LDW"), ("EW_LDW", "EW_MATH"), ("EW_MATH", "EW_PEMPTY"),
               ("EW_S", "EW_PEMPTY"), ("EW_PEMPTY", "EW_DONE"), ("EW_DONE", "MMA23"),
               ("VG_START", "VG_DONE"), ("VG_START", "VG_ISSUED"), ("VG_ISSUED", "VG_DONE"), ("VG_DONE", "MMA1"),
               ("TMA", "EW_Y")]:
    dd = t[lo:hi, EV.index(b_)] - t[lo:hi, EV.index(a_)]
    print("%10s -> %-10s median %7d" % (a_, b_, np.median(dd)))

ew = full[lo:hi, 16:32]
print("per-EW-warp arrival on p_full relative to EW warp 0 (rows = tiles, cols = EW warps 0..15):")
for i in range(ew.shape[0]):
    print("%4d " % (lo + i) + " ".join("%5d" % (ew[i, j] - ew[i, 0]) for j in range(16)))
print("median lag per warp:", [int(np.median(ew[:, j] - ew[:, 0])) for j in range(16)])
