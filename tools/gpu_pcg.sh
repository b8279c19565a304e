#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for sv in 0 1; do
  timeout 300 python tools/perf_c2.py 512,512,512 16 200000 10 $sv >> gpurun_out/pcg_perf.log 2>&1
  echo "rc=$?" >> gpurun_out/pcg_perf.log
done
timeout 300 python tools/perf_c2.py 100,100,100 5 20000 10 0 >> gpurun_out/pcg_perf.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
