#!/bin/bash
# v10: GPU tests (split PCG under sharding), the P = 1 NCCL sharded bench again, then the ncu
# captures of the other configurations
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v10.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_v10.log
timeout 600 python bench.py --nccl-p1 --steps 50 > gpurun_out/bench_p1_v10.json 2> gpurun_out/bench_p1_v10.err
echo "p1 rc=$?" >> gpurun_out/bench_p1_v10.err
bash tools/gpu_ncu_cfgs.sh
