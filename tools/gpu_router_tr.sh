#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
timeout 300 python -m pytest tests/test_gpu_router_fused.py tests/test_gpu_engine.py -m gpu -q > gpurun_out/router_pytest.log 2>&1; echo rc=$? >> gpurun_out/router_pytest.log
timeout 300 python tools/timeline.py --batch 64 --router-backend fused > gpurun_out/timeline_b64_fused5.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu --batch 16 > gpurun_out/ab_new_b16_$rep.log 2>&1
  PS_LIB_PATH=tools/micro/libpolar_pretr.so timeout 600 python bench.py --no-cpu --batch 16 > gpurun_out/ab_old_b16_$rep.log 2>&1
  for b in 32 64; do
    timeout 600 python bench.py --no-cpu --batch $b --router-backend fused > gpurun_out/ab_fused_b${b}_$rep.log 2>&1
    timeout 600 python bench.py --no-cpu --batch $b --router-backend cublas > gpurun_out/ab_cublas_b${b}_$rep.log 2>&1
  done
done
