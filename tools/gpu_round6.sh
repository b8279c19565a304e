#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for d in 1000 4096; do timeout 30 ./tools/probes/chol_trace $d 2; done > gpurun_out/chol_trace.log 2>&1
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 > gpurun_out/perf_c2.log 2>&1
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bucket_syrk|k_ttm_last|k_bucket_contract" -c 3 -o gpurun_out/prof_gram python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu_gram.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_gram.log
