mkdir -p gpurun_out
python tools/gg_sweep2.py > gpurun_out/gg_sweep2.log 2>&1
python tools/kbench.py --trace > gpurun_out/gg_trace_default.log 2>&1
python tools/kbench.py --trace --stages 7 --target 148 > gpurun_out/gg_trace_s7_148.log 2>&1
