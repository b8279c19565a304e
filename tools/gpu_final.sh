#!/bin/bash
# round-end artifacts: full bench (ours + CPU baseline), reference arm, launch list,
# ncu --set full of the top C2 kernels and of the C4 kernels
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:^k_pcg$|k_ttm_last3|k_vech_bucket2|k_ttm_mid3|k_vech_contract2" -c 5 \
  -o gpurun_out/c2_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c2_ncu_full.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/c2_ncu_full.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_c4_dfib|k_c4_dslab" -c 2 \
  -o gpurun_out/c4_full python bench.py --workload c4 --steps 1 --warmup 3 --c4-s 1e7 > gpurun_out/c4_ncu_full.log 2>&1
echo "ncu3 rc=$?" >> gpurun_out/c4_ncu_full.log
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --c4-s 1e5,1e6,1e7 > gpurun_out/c4.json 2> gpurun_out/c4.err
timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err
