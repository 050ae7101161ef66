#!/bin/bash
# A/B of two builds (libnef_cur.so, libnef_prev.so) on nef_fit timings (interleaved, 2 rounds).
cfg=${1:-c5}
for r in 1 2; do
  for v in cur prev; do
    NEF_LIB=paper_2602_02759_b200/libnef_$v.so python scripts/time_modes.py --config $cfg 2>/dev/null | grep "fit iters=4" | sed "s/^/$v /"
  done
done
