#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "draws or c4" tests/test_gpu_c4.py > gpurun_out/pytest_draw.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_draw.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --c4-s 1e5,1e6,1e7 > gpurun_out/c4.json 2> gpurun_out/c4.err
