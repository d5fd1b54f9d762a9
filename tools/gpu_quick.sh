#!/bin/bash
# GPU check: parity tests, bench, per-kernel launch lists of one polar and one dense step.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
timeout 600 python tools/kbench.py --only sel > gpurun_out/kbench.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_polar.csv python tools/profile_step.py > gpurun_out/prof_polar.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_dense.csv python tools/profile_step.py --mode dense > gpurun_out/prof_dense.log 2>&1
python tools/launch_summary.py gpurun_out/launches_polar.csv gpurun_out/launches_dense.csv > gpurun_out/launch_summary.txt 2>&1
