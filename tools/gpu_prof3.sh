#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/perf1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_vech_bucket|k_vech_contract|k_bucket_h|k_ttm_last|k_ttm_mid|k_rhs" -c 8 -o gpurun_out/gram_full python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
