#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
for rep in 1 2; do
  for b in 16 32; do
    timeout 600 python bench.py --no-cpu --batch $b > gpurun_out/ab_def_b${b}_$rep.log 2>&1
    PS_GG_TARGET=264 timeout 600 python bench.py --no-cpu --batch $b > gpurun_out/ab_t264_b${b}_$rep.log 2>&1
  done
done
