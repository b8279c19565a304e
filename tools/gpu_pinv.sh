#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "spd_solve" > gpurun_out/pytest_pinv.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pinv.log
timeout 900 python tools/c3_probe.py 0 3 > gpurun_out/c3_exact.log 2>&1
echo "rc=$?" >> gpurun_out/c3_exact.log
