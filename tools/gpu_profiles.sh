#!/bin/bash
# Round profile capture: per-kernel launch lists of one polar / one dense
# OPT-6.7B B=64 decode step, and one `ncu --set full` capture per hot kernel
# (SHA tensor-core kernel, top-k/union, gathered UP/DOWN GEMMs, head router).
# Numbers printed under ncu are never bench values.
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_polar.csv \
  python tools/profile_step.py > gpurun_out/prof_polar.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_dense.csv \
  python tools/profile_step.py --mode dense > gpurun_out/prof_dense.log 2>&1
python tools/launch_summary.py gpurun_out/launches_polar.csv gpurun_out/launches_dense.csv > gpurun_out/launch_summary.txt 2>&1
# layer 1 (sparse heads) of a 3-layer model: skip layer 0's kernels with -s
timeout 900 $NCU --set full --import-source on -k regex:sha_mma -s 1 -c 1 -o gpurun_out/full_sha -f \
  python tools/profile_step.py --layers 3 > gpurun_out/ncu_full_sha.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:"topk_rows|head_router|gather_gemm" -c 4 -o gpurun_out/full_sel_gg -f \
  python tools/profile_step.py --layers 2 > gpurun_out/ncu_full_sel_gg.log 2>&1
ls -la gpurun_out | tail -20
