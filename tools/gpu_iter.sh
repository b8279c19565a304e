#!/bin/bash
# tests + C2 perf + launch list (ncu only after the plain run succeeded)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 10 0 > gpurun_out/perf.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu.log 2>&1
echo "rc=$?" >> gpurun_out/perf.log
