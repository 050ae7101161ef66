#!/bin/bash
# One GPU iteration: tc parity tests, per-update timings of c5/c3, pipeline traces of c5.
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python scripts/time_updates.py --config c5 --policies 0 > gpurun_out/tu_c5.log 2>&1
python scripts/time_updates.py --config c3 --policies 0 > gpurun_out/tu_c3.log 2>&1
for e in 0 2; do python scripts/trace_pipeline.py --config c5 --ell $e > gpurun_out/trace_c5_$e.log 2>&1; done
