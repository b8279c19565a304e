#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err
echo "c3 rc=$?" >> gpurun_out/c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_c4_dfib|k_gemm_tn" -c 4 \
  -o gpurun_out/c4_full python bench.py --workload c4 --steps 1 --warmup 3 --c4-s 1e7 > gpurun_out/c4_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/c4_ncu_full.log
