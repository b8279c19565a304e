#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 5 0 20000 > gpurun_out/perf_fsk.log 2>&1
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 5 0 0 >> gpurun_out/perf_fsk.log 2>&1
