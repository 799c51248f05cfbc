
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1600 -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_bounce|k_shade" -s 40 -c 4 -o gpurun_out/prof_r1a $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
