#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_factor_sketch.py -x -q > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 2 0 20000 > gpurun_out/perf_fsk.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_fsk.csv python tools/perf_c2.py 512,512,512 16 200000 2 0 20000 > gpurun_out/ncu_fsk.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fsk.log
