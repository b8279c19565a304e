#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
echo "bench rc=$?" >> gpurun_out/bench_q.err
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_ttm_rowsq|k_ttm_last3<" -c 3 -o gpurun_out/rowloss python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/ncu_rowloss.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_rowloss.log
