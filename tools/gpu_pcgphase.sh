#!/bin/bash
mkdir -p gpurun_out
RTB_PCG_PROF=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 4 > gpurun_out/pcgphase.log 2>&1
echo "rc=$?" >> gpurun_out/pcgphase.log
