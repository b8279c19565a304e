mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 300 python bench.py --steps 20 --warmup 3 --c2-only --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err || tail -20 gpurun_out/b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --c2-only > gpurun_out/ll.log 2>&1; echo ncu rc=$?
