#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c3_launches.csv python tools/c3_probe.py 0 1 > gpurun_out/c3_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/c3_ncu.log
