# Full ncu capture of the three dominant kernels (one launch each, second
# vertex of the second render) on the bench configuration at 2 spp.
mkdir -p gpurun_out
python profiles/scripts/prof_render.py 2 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_shadow_ww|k_trace_closest_ww|k_shade" -s 6 -c 3 -o gpurun_out/prof_r1g python profiles/scripts/prof_render.py 2 1 > gpurun_out/ncu_full_g.log 2>&1
echo full_rc=$?
