#!/bin/bash
# Diagnostics: in-graph attribution, top-k phase trace, chained vs split MLP.
mkdir -p gpurun_out
timeout 300 python tools/topk_trace.py > gpurun_out/topk_trace.log 2>&1
timeout 600 python tools/attrib.py --batch 64 > gpurun_out/attrib_b64.log 2>&1
timeout 600 python tools/chain_bench.py --batches 1,16,64,128,256 > gpurun_out/chain_bench.log 2>&1
timeout 600 python tools/chain_bench.py --router --batches 1,16,64,128,256 > gpurun_out/chain_bench_router.log 2>&1
timeout 600 python tools/attrib.py --batch 1 > gpurun_out/attrib_b1.log 2>&1
