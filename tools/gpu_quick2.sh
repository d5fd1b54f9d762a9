#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
timeout 300 python tools/gg_gap.py > gpurun_out/gg_gap.log 2>&1
