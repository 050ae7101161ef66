"""Join ncu's per-SASS stall samples (--page source --csv --print-source sass) with the
cubin's line table (nvdisasm --print-line-info) to get stall samples per CUDA source line.

usage: ncu_stalls_by_line.py report.ncu-rep kernel.cubin mangled_kernel_name [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
samples = []
for r in rows[2:]:
    try:
        samples.append((int(r[0], 16), int(r[i_s] or 0), r[1]))
    except (ValueError, IndexError):
        pass
base = min(a for a, _, _ in samples)
txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin], capture_output=True, text=True).stdout
line_of = {}
cur, inside = None, False
for l in txt.split("\n"):
    s = l.strip()
    if s.startswith(".text."):
        inside = s == ".text." + fn + ":"
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2)
        if m.group(3):   # attribute inlined helpers to their call site in the kernel body
            cur = m.group(3).split("/")[-1] + ":" + m.group(4) + " <- " + cur
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
tot = 0
for a, s, _ in samples:
    agg[line_of.get(a - base, "?")] += s
    tot += s
print("total samples", tot)
for k, v in agg.most_common(top):
    print("%7d %5.1f%%  %s" % (v, 100.0 * v / tot, k))
