#!/bin/bash
# Round artifacts of one code state (TAG): GPU tests, the default bench (all configs + CPU
# baseline), the reference arm, the C2 ncu launch list and one ncu --set full capture of each
# top C2 kernel. Each ncu pass runs after the same command exited 0 without ncu.
TAG=${1:-cur}
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_full_$TAG.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.err
bash tools/gpu_artifacts.sh $TAG
