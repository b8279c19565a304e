#!/bin/bash
# PCG phase profile at C2 for several slice prefetch depths, then the C1 golden test
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for A in 1 2 3; do
  touch paper_2107_10654_b200/csrc/k_pcg.cu
  RTB_NVCC_EXTRA="-DRTB_PCG_AHEAD=$A" python -m paper_2107_10654_b200.build > /dev/null
  echo "== ahead $A" >> gpurun_out/pcg_ahead.log
  RTB_PCG_PROF=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 0 >> gpurun_out/pcg_ahead.log 2>&1
done
touch paper_2107_10654_b200/csrc/k_pcg.cu
python -m paper_2107_10654_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -k "golden_c1 or pcg" > gpurun_out/pytest_k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_k.log
