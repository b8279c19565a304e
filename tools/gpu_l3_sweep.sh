#!/bin/bash
# k_ttm_last3 chunk width / ring depth sweep (perf_c2 ttm_last_loss family time)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/l3_sweep.log
for cfg in "32 3" "32 4" "48 2" "64 2"; do
  set -- $cfg
  touch paper_2107_10654_b200/csrc/k_ttm.cu
  RTB_NVCC_EXTRA="-DRTB_L3BK=$1 -DRTB_L3ST=$2" python -m paper_2107_10654_b200.build > /dev/null
  echo "== BK=$1 ST=$2" >> gpurun_out/l3_sweep.log
  timeout 300 python tools/perf_c2.py 512,512,512 16 200000 8 0 2>&1 | grep -E "sweeps/s|ttm_last_loss" >> gpurun_out/l3_sweep.log
done
touch paper_2107_10654_b200/csrc/k_ttm.cu
python -m paper_2107_10654_b200.build > /dev/null
