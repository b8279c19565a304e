#!/bin/bash
# packed vs blocks PCG: GPU tests touching PCG, then perf_c2 both ways
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/pcg_ab.log
echo "== packed" >> gpurun_out/pcg_ab.log
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 10 0 2>&1 | grep -E "sweeps/s|pcg  |sketch" >> gpurun_out/pcg_ab.log
echo "== blocks" >> gpurun_out/pcg_ab.log
RTB_PCG_BLOCKS=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 10 0 2>&1 | grep -E "sweeps/s|pcg  |sketch" >> gpurun_out/pcg_ab.log
