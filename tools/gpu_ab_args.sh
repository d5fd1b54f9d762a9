#!/bin/bash
# A/B of bench.py flag sets on one box, alternating:
#   bash tools/gpu_ab_args.sh "--batch 1" "--batch 1 --concurrent-head-router" ...
mkdir -p gpurun_out
rm -f gpurun_out/ab_arg*.log
i=0
for rep in 1 2; do
  i=0
  for args in "$@"; do
    i=$((i+1))
    timeout 600 python bench.py --no-cpu $args > gpurun_out/ab_arg${i}_${rep}.log 2>&1
    echo "arg$i = $args" > gpurun_out/ab_arg${i}.txt
  done
done
