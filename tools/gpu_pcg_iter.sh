#!/bin/bash
# PCG iteration check: the solve's parity tests, the sweep-execution tests, the PCG phase
# profile and a short C2 bench (no CPU baseline).
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_parity.py -x -q -k "pcg or graph or c2" > gpurun_out/pytest_pcg.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pcg.log
RTB_PCG_PROF=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 6 0 > gpurun_out/pcg_prof.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --c2-only --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err || tail -20 gpurun_out/b.err
