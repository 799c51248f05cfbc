mkdir -p gpurun_out
python profiles/scripts/prof_render.py 2 1 > gpurun_out/prof_render.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_shadow_ww|k_trace_closest_ww" -s 4 -c 2 -o gpurun_out/prof_r1e python profiles/scripts/prof_render.py 2 1 > gpurun_out/ncu_full_e.log 2>&1
echo full_rc=$?
