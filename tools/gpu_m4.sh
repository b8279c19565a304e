#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err
echo "c3 rc=$?" >> gpurun_out/c3.err
