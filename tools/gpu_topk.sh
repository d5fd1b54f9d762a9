mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/topk_probe.py > gpurun_out/topk_probe.log 2>&1
python tools/topk_trace.py > gpurun_out/topk_trace.log 2>&1
