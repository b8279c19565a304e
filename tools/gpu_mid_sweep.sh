#!/bin/bash
# k_ttm_mid3 chunk rows / ring depth sweep (perf_c2 ttm_mid family time)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/mid_sweep.log
for cfg in "32 4" "64 2" "32 5" "16 8"; do
  set -- $cfg
  touch paper_2107_10654_b200/csrc/k_ttm.cu
  RTB_NVCC_EXTRA="-DRTB_MIDKB=$1 -DRTB_MIDST=$2" python -m paper_2107_10654_b200.build > /dev/null
  echo "== KB=$1 ST=$2" >> gpurun_out/mid_sweep.log
  timeout 300 python tools/perf_c2.py 512,512,512 16 200000 8 0 2>&1 | grep -E "sweeps/s|ttm_mid" >> gpurun_out/mid_sweep.log
done
touch paper_2107_10654_b200/csrc/k_ttm.cu
python -m paper_2107_10654_b200.build > /dev/null
