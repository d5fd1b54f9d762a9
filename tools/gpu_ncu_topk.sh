mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"topk_rows" -c 1 \
  -o gpurun_out/topk_full -f python tools/profile_step.py --layers 2 > gpurun_out/ncu_topk.log 2>&1
