#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/c3_probe.py 0 3 > gpurun_out/c3_exact.log 2>&1
echo "rc=$?" >> gpurun_out/c3_exact.log
timeout 600 python tools/c3_probe.py 50000 3 > gpurun_out/c3_fs.log 2>&1
echo "rc=$?" >> gpurun_out/c3_fs.log
