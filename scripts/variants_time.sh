#!/bin/bash
# Time several builds of libnef (paper_2602_02759_b200/libnef_<tag>.so) on one config (diagnostics).
cfg=$1; shift
cp paper_2602_02759_b200/libnef.so /tmp/libnef_keep.so
for r in 1 2; do
  for v in "$@"; do
    cp paper_2602_02759_b200/libnef_$v.so paper_2602_02759_b200/libnef.so
    python scripts/time_updates.py --config $cfg --policies 0 --reps 5 2>/dev/null | sed "s/^/$v /"
  done
done
cp /tmp/libnef_keep.so paper_2602_02759_b200/libnef.so
