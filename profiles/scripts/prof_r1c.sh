mkdir -p gpurun_out
python profiles/scripts/prof_render.py 2 1 > gpurun_out/prof_render.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_shadow|k_resolve|k_nee" -s 9 -c 3 -o gpurun_out/prof_r1c python profiles/scripts/prof_render.py 2 1 > gpurun_out/ncu_full_c.log 2>&1
echo full_rc=$?
