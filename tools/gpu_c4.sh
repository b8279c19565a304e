#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_c4.py -x -q > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --c4-s 1e5,1e6,1e7 > gpurun_out/c4.json 2> gpurun_out/c4.err
echo "c4 rc=$?" >> gpurun_out/c4.err
