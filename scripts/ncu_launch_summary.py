"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total and mean device time, share of all libnef kernels and of everything.

    python scripts/ncu_launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6))
ours = {k: v for k, v in agg.items() if k.startswith(("nef::", "tc::", "void tc::", "void nef::"))}
tot_ours = sum(sum(v) for v in ours.values())
tot_all = sum(sum(v) for v in agg.values())
print("# %s: %d launches, %.3f ms total; libnef kernels %d launches, %.3f ms" % (
    path, sum(len(v) for v in agg.values()), tot_all, sum(len(v) for v in ours.values()), tot_ours))
print("# (cold-cache, serialised ncu times: compare shares, not absolutes; non-libnef kernels = "
      "torch input generation outside the timed region)")
print("%-8s %12s %12s %10s  %s" % ("launches", "total_ms", "mean_ms", "share_nef", "kernel"))
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    share = "%.4f" % (sum(v) / tot_ours) if k in ours else "-"
    print("%-8d %12.4f %12.5f %10s  %s" % (len(v), sum(v), sum(v) / len(v), share, k[:110]))
