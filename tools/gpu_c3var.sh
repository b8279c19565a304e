mkdir -p gpurun_out
for v in base RTB_C3_NORHS RTB_C3_NOBLK; do
  if [ $v = base ]; then E=""; else E="$v=1"; fi
  env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_vech_contract3 --log-file gpurun_out/c3_$v.csv python tools/perf_c2.py 512,512,512 16 200000 2 > gpurun_out/c3_$v.log 2>&1
  echo $v; grep contract3 gpurun_out/c3_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
done
