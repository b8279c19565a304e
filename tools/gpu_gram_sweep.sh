#!/bin/bash
# k_vech_bucket2 / k_vech_contract2 chunk sweep (perf_c2 gram family time)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/gram_sweep.log
for cfg in "32 32" "40 32" "32 64" "40 64" "36 48"; do
  set -- $cfg
  touch paper_2107_10654_b200/csrc/k_gram.cu
  RTB_NVCC_EXTRA="-DRTB_KCB=$1 -DRTB_KCC=$2" python -m paper_2107_10654_b200.build > /dev/null
  echo "== KCB=$1 KCC=$2" >> gpurun_out/gram_sweep.log
  timeout 300 python tools/perf_c2.py 512,512,512 16 200000 8 0 2>&1 | grep -E "sweeps/s|gram  " >> gpurun_out/gram_sweep.log
done
touch paper_2107_10654_b200/csrc/k_gram.cu
python -m paper_2107_10654_b200.build > /dev/null
