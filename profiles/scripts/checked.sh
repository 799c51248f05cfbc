# Checked build in place of compute-sanitizer (closed on this GPU pool: runs
# under it have left GPUs needing a reset). libmcg compiled with
# -DMCG_CHECKS=1: every index the hot path computes -- VM operand-stack slots
# and program counter, traversal stack depth, cache cell/slot indices,
# texel coordinates, the sort permutation, path ids, shadow-queue slots -- is
# bounds-checked on the device; a failure prints the check and traps, so the
# launch and the test driving it fail. Runs the sanitizer workload
# (every kernel family once) and the whole -m gpu suite on the checked build.
set -u
mkdir -p gpurun_out
[ -f paper_2305_07238_b200/_lib/exp_checked/libmcg.so ] || bash profiles/scripts/build_variant.sh checked "-DMCG_CHECKS=1"
export MCG_LIB_PATH=paper_2305_07238_b200/_lib/exp_checked/libmcg.so
timeout 600 python profiles/scripts/sanitize.py > gpurun_out/checked_workload.log 2>&1
echo "workload rc=$?" >> gpurun_out/checked_workload.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/checked_tests.log
grep -h "MCG_CHECK failed" gpurun_out/checked_workload.log gpurun_out/checked_tests.log | head -20 > gpurun_out/checked_failures.txt
echo "check failures: $(wc -l < gpurun_out/checked_failures.txt)"
