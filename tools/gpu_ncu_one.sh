# one ncu --set full capture of the kernels matching $1 in a short C2 run (tools/perf_c2.py)
mkdir -p gpurun_out
timeout 300 python tools/perf_c2.py 512,512,512 16 200000 2 > gpurun_out/perf.log 2>&1 || { tail -5 gpurun_out/perf.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -c ${2:-1} -o gpurun_out/one python tools/perf_c2.py 512,512,512 16 200000 2 > gpurun_out/ncu_one.log 2>&1
echo "ncu rc=$?"
