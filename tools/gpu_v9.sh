#!/bin/bash
# v9 check: GPU tests (with the one-rank NCCL callback test), the sharded code path at P = 1
# behind a one-rank NCCL group, and the default headline for comparison.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v9.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_v9.log
timeout 600 python bench.py --nccl-p1 --steps 50 > gpurun_out/bench_p1_v9.json 2> gpurun_out/bench_p1_v9.err
echo "p1 rc=$?" >> gpurun_out/bench_p1_v9.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 3 --c2-only --no-cpu-baseline > gpurun_out/bench_torchrun1_v9.json 2> gpurun_out/bench_torchrun1_v9.err
echo "torchrun rc=$?" >> gpurun_out/bench_torchrun1_v9.err
