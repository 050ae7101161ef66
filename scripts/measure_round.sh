#!/bin/bash
# End-of-round measurements on one B200 (run under gpurun from the repo root):
#   scripts/measure_round.sh OUTDIR
# GPU suite, smoke, bench.py lines of every configuration (value, roofline, cpu_baseline, e2e),
# the reference arm on c5, ncu launch lists of the bench command (c2-c5) and one `ncu --set full`
# capture of a streaming launch per configuration (each ncu run only after the same command has
# exited 0 without ncu).  Summaries go to OUTDIR; the .ncu-rep files too (scratch).
set -u
out=${1:-gpurun_out/final}
mkdir -p "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > "$out/smi.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -q -rs > "$out/gpu_tests.txt" 2>&1; echo "exit $?" >> "$out/gpu_tests.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.txt" 2>&1; echo "smoke exit $?" >> "$out/smoke.txt"
for c in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
timeout 600 python bench.py --impl reference > "$out/bench_ref_c5.json" 2> "$out/bench_ref_c5.err"
for c in c2 c3 c4 c5; do
  args="--config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  if timeout 600 python bench.py $args > "$out/plain_$c.json" 2>&1; then
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file "$out/launches_$c.csv" python bench.py $args > "$out/ncu_launches_$c.log" 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 4 -c 1 \
      -o "$out/full_$c" python bench.py $args > "$out/ncu_full_$c.log" 2>&1
  fi
done
echo done > "$out/DONE"
