mkdir -p gpurun_out
for s in 3 4 6 9 12; do timeout 60 python tools/chain_trace.py 1 $s | grep -E "stages|first_stage|last_ph0|first_flag|end "; done > gpurun_out/chain_stages.log 2>&1
