# ncu of the probe kernel after the head/tail split (v4 and the pipelined v5,
# lookup-all launch on the 1e7x10 table) and of the v2 random-read
# calibration (64 B and 128 B accesses): DRAM bytes, L2 hit rate, DRAM
# throughput. Explains what bounds a random cell probe.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed
for v in 4 10; do
  python profiles/scripts/probe_one.py $v 8 > /dev/null 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:k_probe_bench -s 1 -c 1 --csv python profiles/scripts/probe_one.py $v 8 > gpurun_out/ncu_probe_k_v$v.csv 2>&1
  echo v${v}_rc=$?
done
[ -n "$WITH_RAND" ] && ncu --metrics $M --clock-control none -k regex:k_rand --csv ./profiles/scripts/rand_read2 > gpurun_out/ncu_rand_read2.csv 2>&1
echo rr_rc=$?
