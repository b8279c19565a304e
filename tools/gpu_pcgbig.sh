#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "pcg" > gpurun_out/pytest_pcg.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pcg.log
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err
echo "c3 rc=$?" >> gpurun_out/c3.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
