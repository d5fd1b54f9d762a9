#!/bin/bash
# Same-box A/B of the in-tree library against tools/micro/libpolar_$VAR.so
# on the default bench path (B=64) and B=16, alternating.
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
for rep in 1 2 3; do
  for b in ${AB_BATCHES:-64 16}; do
    timeout 600 python bench.py --no-cpu --batch $b --union-handoff off > gpurun_out/ab_new_b${b}_$rep.log 2>&1
    PS_LIB_PATH=tools/micro/libpolar_${VAR:-prehandoff}.so timeout 600 python bench.py --no-cpu --batch $b --union-handoff off > gpurun_out/ab_old_b${b}_$rep.log 2>&1
  done
done
