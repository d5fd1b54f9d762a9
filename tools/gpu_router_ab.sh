#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
timeout 600 python -m pytest tests/test_gpu_router_fused.py -m gpu -x -q > gpurun_out/rab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rab_pytest.log
timeout 300 python tools/timeline.py --batch 64 --router-backend fused > gpurun_out/timeline_b64_fused2.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu --batch 64 > gpurun_out/ab_cublas64_$rep.log 2>&1
  timeout 600 python bench.py --no-cpu --batch 64 --router-backend fused > gpurun_out/ab_fusednew64_$rep.log 2>&1
  PS_LIB_PATH=tools/micro/libpolar_head.so timeout 600 python bench.py --no-cpu --batch 64 --router-backend fused > gpurun_out/ab_fusedold64_$rep.log 2>&1
  timeout 600 python bench.py --no-cpu --batch 16 > gpurun_out/ab_new16_$rep.log 2>&1
  PS_LIB_PATH=tools/micro/libpolar_head.so timeout 600 python bench.py --no-cpu --batch 16 > gpurun_out/ab_old16_$rep.log 2>&1
done
