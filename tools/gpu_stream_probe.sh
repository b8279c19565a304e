#!/bin/bash
mkdir -p gpurun_out
RTB_TTM_STREAM_ONLY=1 timeout 300 python tools/probes/ttm_stream_probe.py > gpurun_out/sp_plain.log 2>&1 && \
RTB_TTM_STREAM_ONLY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_ttm_mid2 -c 3 --csv --log-file gpurun_out/stream_probe.csv python tools/probes/ttm_stream_probe.py > gpurun_out/sp.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_ttm_mid2 -c 3 --csv --log-file gpurun_out/stream_full.csv python tools/probes/ttm_stream_probe.py >> gpurun_out/sp.log 2>&1
