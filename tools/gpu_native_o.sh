#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
for rep in 1 2; do
  for b in ${AB_BATCHES:-64 16 1}; do
    timeout 600 python bench.py --no-cpu --batch $b > gpurun_out/ab_cublas_b${b}_$rep.log 2>&1
    PS_NATIVE_TAGS=gg_o timeout 600 python bench.py --no-cpu --batch $b > gpurun_out/ab_nativeo_b${b}_$rep.log 2>&1
  done
done
