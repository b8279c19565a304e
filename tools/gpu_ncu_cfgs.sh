#!/bin/bash
# ncu --set full of the top kernels of the other configurations (one launch each), each after
# the same command exited 0 without ncu:
#   C2 perf mode (sketched factor updates: the TMA fiber gather k_fsk_accum3, k_fsk_rows),
#   C3 (order-4 bucketed Gram, large-d PCG with the order-4 DMMA matvec),
#   C4 (Kronecker draws + fiber gather / SYRK),
#   C5 one-GPU share (rank-32 bucket kernel, F3 projection, large-d PCG).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
NCU="ncu --set full --clock-control none --import-source on"
run() {  # name regex count cmd...
  local name=$1 rx=$2 cnt=$3; shift 3
  timeout 600 "$@" > gpurun_out/cfg_$name.log 2>&1 || { echo "$name plain rc=$?"; return; }
  timeout 1500 $NCU -k "regex:$rx" -c $cnt -f -o /tmp/cfg_$name "$@" > gpurun_out/ncu_cfg_$name.log 2>&1
  echo "$name ncu rc=$?"
  # the reports (with source) are too big to travel: summarise on the box
  (echo "# ncu --set full --clock-control none, one launch per kernel: $*"
   python tools/ncu_summary.py /tmp/cfg_$name.ncu-rep; echo
   python tools/ncu_pipe_summary.py /tmp/cfg_$name.ncu-rep) > gpurun_out/ncu_cfg_$name.txt 2>&1
}
# skip the first launches (cold) where the kernel runs once per sweep: -c counts matches in order
run c2perf "k_fsk_accum3|k_fsk_rows|k_fsk_reduce" 6 python tools/perf_c2.py 512,512,512 16 200000 2 0 20000
run c3 "k_pcg_dv|k_pcg_t4|k_bucket_h|k_vech_contract|k_ttm_last|k_ttm_mid" 8 python tools/c3_probe.py 0 2
run c4 "k_c4_dfib|k_c4_dslab|k_c4_kr|k_c4_rows|k_draw_eval|k_c4_gram_out" 8 python bench.py --workload c4 --steps 1 --warmup 3 --c4-s 1e7
run c5 "k_vech_bucket6|k_ttm_mid5|k_ttm_last|k_pcg_dv|k_vech_contract3|k_bucket_h4" 8 python tools/c5_probe.py 8 2
