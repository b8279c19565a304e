#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_vech_bucket2|k_vech_contract2|k_pcg$|k_ttm_mid3|k_ttm_last3" -c 5 \
  -o gpurun_out/c2_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c2_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/c2_ncu_full.log
