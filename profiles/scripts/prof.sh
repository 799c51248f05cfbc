# Profiling pass for one build, tagged TAG (replaces the per-checkpoint
# prof_r1*.sh wrappers of round 1):
#   1. the bench line (no ncu)                        gpurun_out/bench_TAG.json
#   2. launch list of one bench step (gpu__time_duration per launch)
#                                                     gpurun_out/launches_TAG.csv
#   3. DRAM bytes per launch over one full bench render  gpurun_out/traffic_TAG.csv
#   4. one --set full capture of NFULL launches matching KRE, after skipping
#      SKIP matches (mid-render: the table is warm) gpurun_out/prof_TAG.ncu-rep
# Usage: bash profiles/scripts/prof.sh TAG [KRE] [SKIP] [NFULL]
# Summaries: python profiles/scripts/summarize.py {launches,traffic,rep} ...
tag=$1
kre=${2:-"k_shade|k_trace_closest_ww|k_shadow_ww|k_lookahead"}
skip=${3:-400}
nfull=${4:-4}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo bench_rc=$?
LCMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
timeout 600 $LCMD > gpurun_out/plain_$tag.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 700 --csv \
    --log-file gpurun_out/launches_$tag.csv $LCMD > gpurun_out/ncu_launch_$tag.log 2>&1
echo launches_rc=$?
timeout 300 python profiles/scripts/prof_render.py 128 1 1 > gpurun_out/traffic_plain_$tag.log 2>&1 && \
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_trace_closest|k_shadow|k_shade|k_primary|k_lookahead" --csv --log-file gpurun_out/traffic_$tag.csv \
    python profiles/scripts/prof_render.py 128 1 1 > gpurun_out/ncu_traffic_$tag.log 2>&1
echo traffic_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $nfull \
    -o gpurun_out/prof_$tag python profiles/scripts/prof_render.py 128 1 1 > gpurun_out/ncu_full_$tag.log 2>&1
echo full_rc=$?
