#!/bin/bash
# A/B over an environment variable: ENV_NAME, ENV_VALUES (space-separated), AB_ARGS as in gpu_ab.sh
mkdir -p gpurun_out
: > gpurun_out/ab_env.log
for v in $ENV_VALUES; do
  echo "#### $ENV_NAME=$v" >> gpurun_out/ab_env.log
  env "$ENV_NAME=$v" bash tools/gpu_ab.sh > /dev/null 2>&1
  cat gpurun_out/ab.log >> gpurun_out/ab_env.log
done
cat gpurun_out/ab_env.log
