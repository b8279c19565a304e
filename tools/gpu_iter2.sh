#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 10 0 > gpurun_out/perf.log 2>&1
RTB_PCG_PROF=1 timeout 300 python tools/probes/noise_probe.py > gpurun_out/noise.log 2>&1
