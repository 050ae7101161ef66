"""Top stall reasons per source line (ncu source page joined with the cubin line table):
ncu_stall_reasons.py report cubin kernel line1 [line2 ...]   (lines of kernels_tc.cu)"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, fn = sys.argv[1:4]
want = set("kernels_tc.cu:" + x for x in sys.argv[4:])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
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
        cur = (m.group(3) or m.group(1)).split("/")[-1] + ":" + (m.group(4) or m.group(2))
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
agg = collections.defaultdict(collections.Counter)
for a, r in data:
    ln = line_of.get(a - base, "?")
    for i in cols:
        try:
            agg[ln][hdr[i]] += int(r[i] or 0)
        except ValueError:
            pass
for ln in sorted(want, key=lambda x: int(x.split(":")[1])):
    tot = sum(agg[ln].values())
    print("%-20s %7d  %s" % (ln, tot, ", ".join("%s %d" % (k[6:], v) for k, v in agg[ln].most_common(4))))
