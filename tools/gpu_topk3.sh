#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_tp.py -m gpu -x -q > gpurun_out/topk3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/topk3_pytest.log
timeout 300 python tools/topk_trace.py > gpurun_out/topk_trace_new.log 2>&1
PS_LIB_PATH=tools/micro/libpolar_oldgemv.so timeout 300 python tools/topk_trace.py > gpurun_out/topk_trace_old.log 2>&1
