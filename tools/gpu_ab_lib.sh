#!/bin/bash
# A/B of the in-tree library against a variant (PS_LIB_PATH) on the same box:
#   bash tools/gpu_ab_lib.sh tools/micro/libpolar_X.so "--batch 64" "--batch 1"
mkdir -p gpurun_out
var=$1; shift
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for args in "$@"; do
  tag=$(echo "$args" | tr -d ' -')
  for rep in 1 2; do
    timeout 600 python bench.py --no-cpu $args > gpurun_out/ab_new_${tag}_$rep.log 2>&1
    PS_LIB_PATH=$var timeout 600 python bench.py --no-cpu $args > gpurun_out/ab_old_${tag}_$rep.log 2>&1
  done
done
