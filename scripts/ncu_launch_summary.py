"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv) per kernel: launches, total / mean device time, share of all libnef
kernels, mean DRAM bytes per launch.

    python scripts/ncu_launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
launch = collections.OrderedDict()
for r in rows[1:]:
    m = launch.setdefault((int(r[ii]), r[ki]), {})
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        v *= scale.get(r[ui], 1e-6)
    elif r[ui] in ("Gbyte", "Mbyte", "Kbyte"):
        v *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}[r[ui]]
    m[r[mi]] = v
agg = collections.defaultdict(list)
for (i, k), m in launch.items():
    agg[k].append(m)
OUR_NAMES = ("sentinel", "pad_rows", "reduce_q_kernel", "update_kernel", "loss_reduce_kernel", "einstep_kernel",
             "fused_ffma_kernel", "fused_tc_kernel")
ours = {k for k in agg if k.startswith(("nef::", "tc::", "void tc::", "void nef::")) or any(n in k for n in OUR_NAMES)}
t = lambda ms: sum(x.get("gpu__time_duration.sum", 0.0) for x in ms)
tot_ours = sum(t(v) for k, v in agg.items() if k in ours)
tot_all = sum(t(v) for v in agg.values())
print("# %s: %d launches, %.3f ms total; libnef kernels %d launches, %.3f ms" % (
    path, len(launch), tot_all, sum(len(v) for k, v in agg.items() if k in ours), tot_ours))
print("# (cold-cache, serialised ncu times: compare shares, not absolutes; non-libnef kernels = "
      "torch input generation outside the timed region)")
print("%-8s %12s %12s %10s %14s %14s  %s" % ("launches", "total_ms", "mean_ms", "share_nef", "dram_rd_B/launch",
                                              "dram_wr_B/launch", "kernel"))
for k, v in sorted(agg.items(), key=lambda x: -t(x[1])):
    share = "%.4f" % (t(v) / tot_ours) if k in ours else "-"
    rd = sum(x.get("dram__bytes_read.sum", 0.0) for x in v) / len(v)
    wr = sum(x.get("dram__bytes_write.sum", 0.0) for x in v) / len(v)
    print("%-8d %12.4f %12.5f %10s %14.4g %14.4g  %s" % (len(v), t(v), t(v) / len(v), share, rd, wr, k[:100]))
