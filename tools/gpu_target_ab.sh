#!/bin/bash
# A/B of the split-K CTA slot target (PS_GG_TARGET) on bench configs.
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu --batch 128 > gpurun_out/ab_def_b128_$rep.log 2>&1
  PS_GG_TARGET=277 timeout 600 python bench.py --no-cpu --batch 128 > gpurun_out/ab_t277_b128_$rep.log 2>&1
  timeout 600 python bench.py --no-cpu --batch 256 > gpurun_out/ab_def_b256_$rep.log 2>&1
  PS_GG_TARGET=138 timeout 600 python bench.py --no-cpu --batch 256 > gpurun_out/ab_t138_b256_$rep.log 2>&1
done
