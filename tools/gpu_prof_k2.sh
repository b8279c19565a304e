#!/bin/bash
# usage: gpu_prof_k2.sh <kernel regex> <outname> [count] -- ncu --set full of a perf_c2 run
mkdir -p gpurun_out
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -c ${3:-1} -o gpurun_out/$2 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu_$2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$2.log
