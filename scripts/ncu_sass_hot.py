"""Top SASS instructions by stall samples within a source-line range of kernels_tc.cu:
ncu_sass_hot.py report cubin kernel first_line last_line [top]"""
import csv
import io
import re
import subprocess
import sys

rep, cubin, fn, l0, l1 = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
top = int(sys.argv[6]) if len(sys.argv) > 6 else 40
import os
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + os.environ.get("NCU_FILTER", "").split(), capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
isamp = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
txt = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin], capture_output=True, text=True).stdout
line_of, cur, inside = {}, None, False
for l in txt.split("\n"):
    s = l.strip()
    if s.startswith(".text."):
        inside = s == ".text." + fn + ":"
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        cur = int(m.group(4) or m.group(2)) if (m.group(3) or m.group(1)).endswith("kernels_tc.cu") else None
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), r))
    except (ValueError, IndexError):
        pass
base = min(a for a, _ in data)
sel = []
for a, r in data:
    ln = line_of.get(a - base)
    if ln is not None and l0 <= ln <= l1:
        samp = int(r[isamp] or 0)
        st = sorted(((int(r[i] or 0), hdr[i][6:]) for i in cols), reverse=True)[:3]
        sel.append((samp, a - base, ln, r[isrc], int(float(r[ie] or 0)), st))
tot = sum(x[0] for x in sel)
print("samples in lines %d-%d: %d" % (l0, l1, tot))
for x in sorted(sel, reverse=True)[:top]:
    print("%6d %6x L%d %-60s exec %9d  %s" % (x[0], x[1], x[2], x[3][:60], x[4], ", ".join("%s %d" % (n, v) for v, n in x[5] if v)))
