#!/bin/bash
# ncu --set full of the C5 core-update solve kernels (tools/c5_probe.py, replicated solve)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/c5_probe.py 8 2 > gpurun_out/cfg_c5.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_pcg_dv|k_pcg_prep|k_vech_blocks" -c 3 -f -o /tmp/cfg_c5core python tools/c5_probe.py 8 2 > gpurun_out/ncu_cfg_c5core.log 2>&1
echo "ncu rc=$?"
(echo "# ncu --set full --clock-control none, one launch per kernel: python tools/c5_probe.py 8 2"
 python tools/ncu_summary.py /tmp/cfg_c5core.ncu-rep; echo
 python tools/ncu_pipe_summary.py /tmp/cfg_c5core.ncu-rep) > gpurun_out/ncu_cfg_c5core.txt 2>&1
