#!/bin/bash
# C4 tests + C4 microbench (+ optional launch list of one s=1e7 step)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_c4.py -x -q > gpurun_out/pytest_c4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c4.log
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --c4-s 1e5,1e6,1e7 > gpurun_out/c4.json 2> gpurun_out/c4.err
echo "c4 rc=$?" >> gpurun_out/c4.err
if [ "$1" = "launches" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c4_launches.csv python bench.py --workload c4 --steps 1 --warmup 0 --c4-s 1e7 > gpurun_out/c4_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/c4_ncu.log
fi
