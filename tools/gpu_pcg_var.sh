# A/B of PCG variants (tools/varlib.sh builds): per-phase ns of CTA 0 (RTB_PCG_PROF)
mkdir -p gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="RTB_LIB_PATH=explib/$v/librtucker_b200.so"; fi
  echo "== $v"
  env $L RTB_PCG_PROF=1 timeout 300 python tools/perf_c2.py 512,512,512 16 200000 3 2>&1 | grep -E "^\[pcg|pcg  " | tail -3
done
