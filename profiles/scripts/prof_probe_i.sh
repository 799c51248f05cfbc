# ncu of the probe kernel: v4 on the 1e7x10 table, v0 on the L2-resident
# 1e5x10 table (lookup-all launch): DRAM bytes, L2 hit rate, warp efficiency.
mkdir -p gpurun_out
python profiles/scripts/probe_one.py 4 8 > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:k_probe_bench -s 1 -c 1 -o gpurun_out/prof_probe_v4_big python profiles/scripts/probe_one.py 4 8 > gpurun_out/ncu_probe_big.log 2>&1
echo big_rc=$?
python profiles/scripts/probe_one.py 0 8 100000 > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:k_probe_bench -s 1 -c 1 -o gpurun_out/prof_probe_v0_small python profiles/scripts/probe_one.py 0 8 100000 > gpurun_out/ncu_probe_small.log 2>&1
echo small_rc=$?
