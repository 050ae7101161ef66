#!/bin/bash
# A/B of two builds (libnef_cur.so, libnef_prev.so) on the per-mode timings of time_modes.py.
cfg=${1:-c5}
for r in 1 2; do
  for v in cur prev; do
    NEF_LIB=paper_2602_02759_b200/libnef_$v.so python scripts/time_modes.py --config $cfg 2>/dev/null | sed "s/^/$v /"
  done
done
