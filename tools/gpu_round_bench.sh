#!/bin/bash
# golden test, full bench (ours + reference arm), launch list, one ncu --set full of the top kernels
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -q -k "golden_c1 or c4 or factor_sketch" > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
./tools/gpu_bench_full.sh
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:^k_pcg$|k_ttm_last3|k_vech_bucket2|k_ttm_mid3|k_vech_contract2" -c 5 -o gpurun_out/top_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_top.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_top.log
