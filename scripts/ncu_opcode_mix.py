"""Executed warp instructions per opcode (and per tile) of the kernel in an ncu report:
ncu_opcode_mix.py report entries_per_launch [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, entries = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
tiles = entries / 8192.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ie, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
mix = collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    s = r[isrc].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op = s.split()[0] if s else "?"
    mix[op.split(".")[0]] += n
tot = sum(mix.values())
print("total warp instr per tile %.0f" % (tot / tiles))
for op, n in mix.most_common(top):
    print("%-12s %7.0f /tile  %5.1f%%" % (op, n / tiles, 100.0 * n / tot))
