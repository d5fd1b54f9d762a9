#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_adapter.py -x -q > gpurun_out/pytest_adapter.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"topk_rows|head_router|layernorm|kv_append" -c 8 \
  -o gpurun_out/sel_full -f python tools/profile_step.py --layers 3 > gpurun_out/ncu_sel.log 2>&1
