#!/bin/bash
# c5 re-measurement after a kernel change (run under gpurun from the repo root):
#   scripts/measure_c5.sh OUTDIR
# GPU suite with the parity-error log, randomized parity sweeps, the c5 bench line, its ncu launch
# list and one ncu --set full capture (summarised here; the report stays on the box).
set -u
out=${1:-gpurun_out/c5}
mkdir -p "$out"
NEF_ERR_LOG="$out/parity_errors.jsonl" timeout 900 python -m pytest tests -m gpu -q > "$out/gpu_tests.txt" 2>&1; echo "exit $?" >> "$out/gpu_tests.txt"
for sd in 7 11 13; do
  echo "seed $sd: $(NEF_RANDOM_CASES=200 NEF_RANDOM_SEED=$sd timeout 400 python -m pytest tests/test_gpu_edges.py -k random -q 2>&1 | tail -1)" >> "$out/random.txt"
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.txt" 2>&1; echo "smoke exit $?" >> "$out/smoke.txt"
timeout 900 python bench.py > "$out/bench_c5.json" 2> "$out/bench_c5.err"
args="--config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 600 python bench.py $args > "$out/plain_c5.json" 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file "$out/launches_c5.csv" python bench.py $args > "$out/ncu_launches_c5.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 4 -c 1 \
    -o "$out/full_c5" python bench.py $args > "$out/ncu_full_c5.log" 2>&1
  python scripts/ncu_launch_summary.py "$out/launches_c5.csv" > "$out/launches_c5.txt" 2>&1
  python scripts/ncu_full_summary.py "$out/full_c5.ncu-rep" > "$out/ncu_full_c5.txt" 2>&1
  rm -f "$out/full_c5.ncu-rep" "$out/launches_c5.csv"
fi
echo done > "$out/DONE"
