#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
for rep in 1 2 3; do
  for b in ${AB_BATCHES:-64 16}; do
    timeout 600 python bench.py --no-cpu --batch $b --union-handoff off > gpurun_out/ab_off_b${b}_$rep.log 2>&1
    timeout 600 python bench.py --no-cpu --batch $b --union-handoff on > gpurun_out/ab_on_b${b}_$rep.log 2>&1
  done
done
timeout 300 python tools/timeline.py --batch 64 > gpurun_out/timeline_b64_off.log 2>&1
