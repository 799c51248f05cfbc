# DRAM bytes per launch of every kernel of ONE full bench render (1920x1080x128,
# cache 1e7x10), averaged per kernel class -> profiles/dram_traffic.json.
mkdir -p gpurun_out
python profiles/scripts/prof_render.py 128 1 1 > gpurun_out/traffic_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_trace_closest|k_shadow|k_shade|k_primary" --csv --log-file gpurun_out/traffic.csv \
    python profiles/scripts/prof_render.py 128 1 1 > gpurun_out/ncu_traffic.log 2>&1
echo traffic_rc=$?
