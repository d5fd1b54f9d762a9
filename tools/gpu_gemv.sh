#!/bin/bash
# B=1 anatomy: the small-batch GEMV alone (new vs HEAD variant), the in-graph
# timeline and launch lists of one polar and one dense step at B = 1.
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --clock-control none"
timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_new.log 2>&1
[ -f tools/micro/libpolar_oldgemv.so ] && PS_LIB_PATH=tools/micro/libpolar_oldgemv.so timeout 300 python tools/gemv_bench.py > gpurun_out/gemv_old.log 2>&1
timeout 300 python tools/timeline.py --batch 1 > gpurun_out/timeline_b1.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_polar_b1.csv \
  python tools/profile_step.py --batch 1 > gpurun_out/prof_polar_b1.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_dense_b1.csv \
  python tools/profile_step.py --batch 1 --mode dense > gpurun_out/prof_dense_b1.log 2>&1
python tools/launch_summary.py gpurun_out/launches_polar_b1.csv gpurun_out/launches_dense_b1.csv > gpurun_out/launch_summary_b1.txt 2>&1
