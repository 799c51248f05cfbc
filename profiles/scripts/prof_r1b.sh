mkdir -p gpurun_out
python profiles/scripts/prof_render.py 2 1 > gpurun_out/prof_render.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bounce|k_shade" -s 12 -c 3 -o gpurun_out/prof_r1b python profiles/scripts/prof_render.py 2 1 > gpurun_out/ncu_full_b.log 2>&1
echo full_rc=$?
