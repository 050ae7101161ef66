"""Attribute SASS instructions of one kernel to source lines (needs a -lineinfo cubin)."""
import collections
import re
import subprocess
import sys

cubin, fn = sys.argv[1], sys.argv[2]
txt = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
cnt = collections.Counter()
cur = None
n = 0
inside = False
for l in txt.split("\n"):
    if re.match(r"^\.?[\w.]*:\s*$", l.strip()) or l.startswith(".text.") or l.startswith("\t.section"):
        if l.strip().startswith(".text." + fn) or l.strip() == fn + ":":
            inside = True
        elif l.startswith(".text.") or l.startswith("\t.section"):
            if inside and n > 0:
                break
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = m.group(1).split("/")[-1] + ":" + m.group(2)
    elif re.search(r"/\*[0-9a-f]{4,}\*/", l):
        cnt[cur] += 1
        n += 1
print("total", n)
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(v, k)
