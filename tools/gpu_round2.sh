#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/perf1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv python tools/perf_c2.py 512,512,512 16 200000 1 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
