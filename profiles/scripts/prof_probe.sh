mkdir -p gpurun_out
for cfg in "0 2" "0 8" "2 8"; do
  set -- $cfg
  python profiles/scripts/probe_one.py $1 $2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none -k regex:k_probe_bench -s 1 -c 1 -o gpurun_out/prof_probe_v$1_b$2 python profiles/scripts/probe_one.py $1 $2 > gpurun_out/ncu_probe_$1_$2.log 2>&1
  echo "cfg $cfg rc=$?"
done
