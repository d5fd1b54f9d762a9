#!/bin/bash
# One GPU session: parity tests, bench, launch list and an ncu capture of the SHA kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python tools/kbench.py > gpurun_out/kbench.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_polar.csv python tools/profile_step.py > gpurun_out/prof_polar.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_dense.csv python tools/profile_step.py --mode dense > gpurun_out/prof_dense.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:sha_decode -c 2 \
  -o gpurun_out/sha_full -f python tools/profile_step.py --layers 4 > gpurun_out/ncu_sha.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gather_gemm -c 4 \
  -o gpurun_out/gg_full -f python tools/profile_step.py --layers 2 > gpurun_out/ncu_gg.log 2>&1
ls -la gpurun_out
