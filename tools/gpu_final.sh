#!/bin/bash
# Round-end validation: GPU tests, smoke, default bench, reference arm.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo "rc=$?" >> gpurun_out/final_ref.log
