#!/bin/bash
# The TP shapes (configs 4 and 5) at TP=1 on one B200: weights cycled over 8
# distinct layer sets, K/V storage aliased (the full caches exceed 180 GB).
mkdir -p gpurun_out
timeout 1200 python bench.py --tp --config opt-66b --batch 256 --ctx 1920 --rho 0.3 --distinct-layers 8 \
  --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_opt66b_tp1.log 2>&1
timeout 1500 python bench.py --tp --config llama-3.1-70b --batch 512 --ctx 8192 --rho 0.625 --distinct-layers 8 \
  --steps 3 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_llama70b_tp1.log 2>&1
