mkdir -p gpurun_out
for b in 1 64 256; do timeout 60 python tools/chain_trace.py $b; done > gpurun_out/chain_trace.log 2>&1
