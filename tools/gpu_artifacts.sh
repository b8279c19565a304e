#!/bin/bash
# Measurement artifacts of one code state (run under gpurun; TAG names the outputs):
#   1. the default bench line (no profiler),
#   2. the ncu launch list of a short bench run (per-launch device times, serialized),
#   3. one ncu --set full capture of each top C2 kernel.
# Each ncu pass runs only after the same command exited 0 without ncu.
TAG=${1:-cur}
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --steps 20 --warmup 3 --no-extra > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
rc=$?; echo "bench rc=$rc" >> gpurun_out/bench_$TAG.err
[ $rc -eq 0 ] || exit $rc
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --c2-only \
  > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/ncu_launch_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_pcg_split|k_ttm_last5|k_vech_bucket5|k_ttm_mid5|k_vech_contract3" -c 5 \
  -f -o /tmp/full_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --c2-only \
  > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_$TAG.log
# the report (with source) is too big to travel with the rest: summarise it on the box
(echo "# ncu --set full --clock-control none, C2 bench, code state $TAG, one launch of each top kernel"
 python tools/ncu_summary.py /tmp/full_$TAG.ncu-rep; echo
 python tools/ncu_pipe_summary.py /tmp/full_$TAG.ncu-rep) > gpurun_out/ncu_top_$TAG.txt 2>&1
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 0 20000 > gpurun_out/perf_c2_fsk_$TAG.txt 2>&1
