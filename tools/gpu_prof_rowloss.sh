#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_ttm_last3" -c 3 -o gpurun_out/rowloss python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/ncu_rowloss.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_rowloss.log
