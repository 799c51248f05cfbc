# Checkpoint l (shade launch bounds, shared-memory probe resolve): bench line, launch list of the same bench command, whole-render
# DRAM traffic per kernel class, one --set full capture of the three
# dominant kernels.
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err
echo bench_rc=$?
LCMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
$LCMD > gpurun_out/plain_l.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1400 -c 500 --csv --log-file gpurun_out/launches_l.csv $LCMD > gpurun_out/ncu_launch_l.log 2>&1
echo launches_rc=$?
bash profiles/scripts/prof_traffic.sh
python profiles/scripts/summarize.py traffic gpurun_out/traffic.csv > gpurun_out/dram_traffic.json
python profiles/scripts/prof_render.py 2 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_shadow_ww|k_trace_closest_ww|k_shade" -s 6 -c 3 -o gpurun_out/prof_r1l python profiles/scripts/prof_render.py 2 1 > gpurun_out/ncu_full_l.log 2>&1
echo full_rc=$?
