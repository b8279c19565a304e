#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/perf_c2.log 2>&1
./tools/gpu_launches.sh
