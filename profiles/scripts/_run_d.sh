mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -q -s -rA > gpurun_out/r2/gpu_tests_d.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2/gpu_tests_d.log
timeout 1200 python bench.py > gpurun_out/r2/bench_d.json 2> gpurun_out/r2/bench_d.err; echo "bench rc=$?" >> gpurun_out/r2/bench_d.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2/bench_ref_d.json 2> gpurun_out/r2/bench_ref_d.err
