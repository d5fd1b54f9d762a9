#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_router_fused.py -m gpu -x -q > gpurun_out/router_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/router_pytest.log
timeout 300 python tools/timeline.py --batch 1 > gpurun_out/timeline_b1_bar.log 2>&1
timeout 300 python tools/timeline.py --batch 16 > gpurun_out/timeline_b16_bar.log 2>&1
timeout 600 python bench.py --no-cpu --batch 1 > gpurun_out/bench_b1_bar.log 2>&1
timeout 600 python bench.py --no-cpu --batch 16 > gpurun_out/bench_b16_bar.log 2>&1
