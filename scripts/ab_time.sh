#!/bin/bash
# A/B timing of two builds of libnef (diagnostics): interleaved runs of time_updates.py.
cfg=${1:-c5}
cp paper_2602_02759_b200/libnef.so /tmp/libnef_cur.so
for r in 1 2; do
  cp /tmp/libnef_cur.so paper_2602_02759_b200/libnef.so
  python scripts/time_updates.py --config $cfg --policies 0 --reps 5 2>/dev/null | sed "s/^/cur /"
  cp paper_2602_02759_b200/libnef_prev.so paper_2602_02759_b200/libnef.so
  python scripts/time_updates.py --config $cfg --policies 0 --reps 5 2>/dev/null | sed "s/^/prev /"
done
cp /tmp/libnef_cur.so paper_2602_02759_b200/libnef.so
