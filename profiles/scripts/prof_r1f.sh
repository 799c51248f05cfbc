# Checkpoint capture: full bench line, launch list of the same command, and
# one --set full capture of the two traversal kernels.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3"
$CMD > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo bench_rc=$?
LCMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
$LCMD > gpurun_out/plain_l.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2400 -c 700 --csv --log-file gpurun_out/launches_f.csv $LCMD > gpurun_out/ncu_launch_f.log 2>&1
echo launches_rc=$?
python profiles/scripts/prof_render.py 2 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_shadow_ww|k_trace_closest_ww|k_shade" -s 5 -c 3 -o gpurun_out/prof_r1f python profiles/scripts/prof_render.py 2 1 > gpurun_out/ncu_full_f.log 2>&1
echo full_rc=$?
