"""A/B timing of library variants through bench.py (diagnostics; one B200 under gpurun):

    python scripts/ab_bench.py OUT.jsonl c5,c3 base=paper_2602_02759_b200/libnef_base.so new= [reps]

Each (config, variant) runs `bench.py --config cN --no-e2e --no-cpu-baseline` with NEF_LIB set to
the variant's library (empty: the default libnef.so), interleaved over `reps` rounds so clock and
power-cap drift hit every variant alike; one JSON line per run is appended to OUT.jsonl and a
summary (median ms per sweep, roofline frac, SM clock) is printed per (config, variant)."""
import json
import os
import statistics
import subprocess
import sys

out, cfgs = sys.argv[1], sys.argv[2].split(",")
variants = []
reps = 2
for a in sys.argv[3:]:
    if "=" in a:
        k, v = a.split("=", 1)
        variants.append((k, v))
    else:
        reps = int(a)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {}
with open(out, "a") as f:
    for r in range(reps):
        for cfg in cfgs:
            for tag, lib in variants:
                env = dict(os.environ)
                if lib:
                    env["NEF_LIB"] = os.path.join(root, lib)
                p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", cfg, "--no-e2e",
                                    "--no-cpu-baseline"], capture_output=True, text=True, env=env, timeout=600)
                line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else "{}"
                try:
                    d = json.loads(line)
                except ValueError:
                    d = {}
                rec = {"cfg": cfg, "variant": tag, "rep": r, "ms": d.get("ms_per_step"),
                       "frac": (d.get("roofline") or {}).get("frac"), "clocks": d.get("clocks"),
                       "rc": p.returncode, "err": p.stderr[-300:] if p.returncode else ""}
                f.write(json.dumps(rec) + "\n")
                f.flush()
                res.setdefault((cfg, tag), []).append(rec)
for (cfg, tag), recs in sorted(res.items()):
    ms = [x["ms"] for x in recs if x["ms"]]
    fr = [x["frac"] for x in recs if x["frac"]]
    mhz = [x["clocks"]["sm_mhz"] for x in recs if x.get("clocks") and x["clocks"].get("sm_mhz")]
    print("%s %-8s ms %s frac %s mhz %s" % (cfg, tag, ("%.4f" % statistics.median(ms)) if ms else None,
                                          ("%.3f" % statistics.median(fr)) if fr else None,
                                          statistics.median(mhz) if mhz else None))
