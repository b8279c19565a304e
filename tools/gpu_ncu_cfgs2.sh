#!/bin/bash
# second pass of tools/gpu_ncu_cfgs.sh: the core-update kernels of C3 and C5 (the first pass's
# launch budget went to the TTM kernels that run first in a sweep)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
NCU="ncu --set full --clock-control none --import-source on"
run() {
  local name=$1 rx=$2 cnt=$3; shift 3
  timeout 1500 $NCU -k "regex:$rx" -c $cnt -f -o /tmp/cfg_$name "$@" > gpurun_out/ncu_cfg_$name.log 2>&1
  echo "$name ncu rc=$?"
  (echo "# ncu --set full --clock-control none, one launch per kernel: $*"
   python tools/ncu_summary.py /tmp/cfg_$name.ncu-rep; echo
   python tools/ncu_pipe_summary.py /tmp/cfg_$name.ncu-rep) > gpurun_out/ncu_cfg_$name.txt 2>&1
}
timeout 600 python tools/c3_probe.py 0 2 > gpurun_out/cfg_c3.log 2>&1 || exit 1
run c3core "k_pcg_dv|k_pcg_t4|k_bucket_h|k_vech_contract|k_vech_bucket|k_gather_draws|k_draw_eval" 7 python tools/c3_probe.py 0 2
timeout 600 python tools/c5_probe.py 8 2 > gpurun_out/cfg_c5.log 2>&1 || exit 1
run c5core "k_pcg_dv|k_pcg_prep|k_vech_expand|k_vech_blocks" 4 python tools/c5_probe.py 8 2
