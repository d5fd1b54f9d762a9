#!/bin/bash
# Round-end validation + refreshed captures: GPU tests, smoke, default bench
# (B=64, CPU baseline), the reference arm, B=1 / B=8 bench lines, the B=1 and
# B=64 in-graph timelines and launch lists.
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --clock-control none"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo "rc=$?" >> gpurun_out/final_ref.log
timeout 600 python bench.py --no-cpu --batch 1 > gpurun_out/final_bench_b1.log 2>&1
timeout 600 python bench.py --no-cpu --batch 8 > gpurun_out/final_bench_b8.log 2>&1
timeout 300 python tools/timeline.py --batch 1 > gpurun_out/final_timeline_b1.log 2>&1
timeout 300 python tools/timeline.py --batch 64 > gpurun_out/final_timeline_b64.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/final_launches_polar_b1.csv \
  python tools/profile_step.py --batch 1 > /dev/null 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/final_launches_dense_b1.csv \
  python tools/profile_step.py --batch 1 --mode dense > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/final_launches_polar_b1.csv gpurun_out/final_launches_dense_b1.csv > gpurun_out/final_launch_summary_b1.txt 2>&1
