#!/bin/bash
# full GPU test suite + default bench (no CPU baseline) + C4 microbench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
echo "bench rc=$?" >> gpurun_out/bench_q.err
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --c4-s 1e5,1e6,1e7 > gpurun_out/c4.json 2> gpurun_out/c4.err
echo "c4 rc=$?" >> gpurun_out/c4.err
