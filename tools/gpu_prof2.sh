#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/pcg_full2 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sym_eigen_warp --launch-skip 4 -c 1 -o gpurun_out/eig_full python tools/perf_c2.py 512,512,512 16 200000 1 >> gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
