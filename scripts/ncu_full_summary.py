"""Key metrics of one kernel in an `ncu --set full` report (roofline evidence, pipe utilisation,
stall reasons): python scripts/ncu_full_summary.py report.ncu-rep [algorithmic_bytes]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
algo = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
keys = [
    "Kernel Name", "Grid Size", "Block Size", "launch__registers_per_thread", "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
]
print("# ncu --set full summary of %s" % rep)
for k in keys:
    if k in d:
        print("%-80s %s %s" % (k, d[k][0], d[k][1]))
rd = float(d["dram__bytes_read.sum"][0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1.0}.get(d["dram__bytes_read.sum"][1], 1.0)
wr = float(d["dram__bytes_write.sum"][0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(d["dram__bytes_write.sum"][1], 1.0)
print("%-80s %.6g" % ("dram bytes (read + write) per launch", rd + wr))
if algo:
    print("%-80s %.6g (traffic / algorithmic = %.3f)" % ("algorithmic bytes per launch", algo, (rd + wr) / algo))
print("# warp stall samples (pc sampling), descending")
st = [(int(float(v[0])), h[33:]) for h, v in d.items()
      if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
tot = sum(x for x, _ in st)
for n, h in sorted(st, reverse=True):
    if n:
        print("%-40s %8d  %5.1f%%" % (h, n, 100.0 * n / tot))
