#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
echo "bench rc=$?" >> gpurun_out/bench_q.err
RTB_PCG_PROF=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 6 0 > gpurun_out/pcg_prof.log 2>&1
