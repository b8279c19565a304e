# A/B of variant builds (tools/varlib.sh): ncu launch times of kernels matching $1 in a short C2 run
mkdir -p gpurun_out
K=$1; shift
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="RTB_LIB_PATH=explib/$v/librtucker_b200.so"; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "regex:$K" --log-file gpurun_out/v_$v.csv python tools/perf_c2.py 512,512,512 16 200000 2 > gpurun_out/v_$v.log 2>&1
  echo "$v: $(grep -v '^==' gpurun_out/v_$v.csv | tail -n +2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
