#!/bin/bash
# Full GPU verification: all -m gpu tests, smoke, bench (every config), launch list + ncu full of c5.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?
for c in c1 c2 c3 c4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c5.json 2> gpurun_out/bench_ref_c5.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled -k regex:'nef::' -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu_l=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 2 -c 1 \
  -o gpurun_out/c5_full -f python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo ncu_f=$?
