#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
timeout 900 python -m pytest tests/test_gpu_union_handoff.py tests/test_gpu_engine.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/handoff_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/handoff_pytest.log
timeout 300 python tools/timeline.py --batch 64 > gpurun_out/timeline_b64_handoff.log 2>&1
for rep in 1 2; do
  for b in 64 16; do
    timeout 600 python bench.py --no-cpu --batch $b --union-handoff off > gpurun_out/ab_off_b${b}_$rep.log 2>&1
    timeout 600 python bench.py --no-cpu --batch $b --union-handoff on > gpurun_out/ab_on_b${b}_$rep.log 2>&1
  done
done
