#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
rm -f gpurun_out/pcg_form.log
for thr in 4.0 0.0; do
  touch paper_2107_10654_b200/csrc/k_pcg.cu
  RTB_NVCC_EXTRA="-DRTB_EIG_ABOVE=$thr" python -m paper_2107_10654_b200.build > /dev/null
  echo "== eig_above=$thr" >> gpurun_out/pcg_form.log
  timeout 300 python tools/perf_c2.py 512,512,512 16 200000 10 0 2>&1 | grep -E "sweeps/s|pcg  |sketch" >> gpurun_out/pcg_form.log
done
touch paper_2107_10654_b200/csrc/k_pcg.cu
python -m paper_2107_10654_b200.build > /dev/null
