#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/perf_c2.py 160,160,160,160 10 500000 2 > gpurun_out/c3.log 2>&1
echo "rc=$?" >> gpurun_out/c3.log
