#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_pcg.csv python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/pcg_full python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
