#!/bin/bash
# launch list (per-kernel device times) of a short perf_c2 run
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/perf1.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/ncu_ll.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_ll.log
