"""Per-source-line executed warp instructions and stall samples of one kernel in an ncu report,
normalised per 64-column tile: ncu_instr_by_line.py report cubin kernel entries_per_launch [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, fn, entries = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
tiles = entries / 8192.0
import os
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + os.environ.get("NCU_FILTER", "").split(), capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iexc = hdr.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in hdr else None
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
        data.append((int(r[0], 16), int(r[ie] or 0), int(r[isamp] or 0),
                     int(float(r[iexc] or 0)) if iexc is not None else 0))
    except (ValueError, IndexError):
        pass
base = min(d[0] for d in data)
ins, smp, exc = collections.Counter(), collections.Counter(), collections.Counter()
for a, n, s, x in data:
    k = line_of.get(a - base, "?")
    ins[k] += n
    smp[k] += s
    exc[k] += x
ti, ts = sum(ins.values()), sum(smp.values())
print("warp instr per tile %.0f   samples %d" % (ti / tiles, ts))
for k, v in ins.most_common(top):
    print("%7.0f instr/tile %5.1f%%   stall %5.1f%%   %s" % (v / tiles, 100 * v / ti, 100 * smp[k] / ts, k))
tx = sum(exc.values())
if tx:
    print("# shared-memory excessive wavefronts (bank conflicts) per tile %.0f, by line" % (tx / tiles))
    for k, v in exc.most_common(8):
        print("%7.0f excess wavefronts/tile %5.1f%%   %s" % (v / tiles, 100 * v / tx, k))
