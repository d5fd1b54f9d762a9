mkdir -p gpurun_out
for d in 0 1 2 3; do echo "== dbg $d"; PS_CHAIN_DBG=$d timeout 60 python tools/chain_trace.py 64 | grep -E "last_ph0|first_flag|end |p0_|fin"; done > gpurun_out/chain_gate.log 2>&1
