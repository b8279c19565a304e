# A/B of runtime env toggles: ncu launch times of kernels matching $1 in a short C2 run, per env setting
mkdir -p gpurun_out
K=$1; shift
for v in base "$@"; do
  if [ $v = base ]; then E=""; else E="$v=1"; fi
  env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "regex:$K" --log-file gpurun_out/e_$v.csv python tools/perf_c2.py 512,512,512 16 200000 2 > gpurun_out/e_$v.log 2>&1
  echo "$v: $(grep -v '^==' gpurun_out/e_$v.csv | tail -n +2 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
  grep -E "final loss" gpurun_out/e_$v.log
done
