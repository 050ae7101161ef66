"""Markdown table of the measured parity errors recorded by the GPU tests (NEF_ERR_LOG JSON lines,
tests/conftest.py::record_err): worst error per test against its bar.
    python scripts/parity_table.py profiles/r02_parity_errors.jsonl"""
import json
import sys

rows = {}
for path in sys.argv[1:]:
    for line in open(path):
        r = json.loads(line)
        key = (r["test"].split("::", 1)[-1], r["what"])
        if key not in rows or r["err"] > rows[key]["err"]:
            rows[key] = r
print("| test | quantity | worst error | bar | margin |")
print("|---|---|---|---|---|")
for (test, what), r in sorted(rows.items(), key=lambda kv: -kv[1]["err"] / kv[1]["bar"]):
    print("| `%s` | %s | %.2e | %.0e | %.1fx |" % (test, what, r["err"], r["bar"], r["bar"] / max(r["err"], 1e-300)))
