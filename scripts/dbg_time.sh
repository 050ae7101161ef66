#!/bin/bash
# Timing experiments with diagnostic kernel switches (NEF_TC_DBG bits; results invalid).
cfg=${1:-c5}
for d in ${DBGS:-0 32 64 128 96 224}; do
  NEF_TC_DBG=$d python scripts/time_updates.py --config $cfg --policies 0 --reps 5 2>/dev/null | sed "s/^/dbg$d /"
done
