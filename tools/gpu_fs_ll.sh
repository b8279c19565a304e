mkdir -p gpurun_out
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 0 20000 > gpurun_out/fs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fs.csv python tools/perf_c2.py 512,512,512 16 200000 3 0 20000 > gpurun_out/fs_ncu.log 2>&1
echo rc=$?
