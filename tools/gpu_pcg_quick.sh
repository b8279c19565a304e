#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
RTB_PCG_PROF=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 0 > gpurun_out/pcg_prof.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "pcg or sketched or golden or sharded" > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
