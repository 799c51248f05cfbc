mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gpu_tests_c.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2/gpu_tests_c.log
bash profiles/scripts/ab.sh "base MCG_LIB_PATH=paper_2305_07238_b200/_lib/exp_base/libmcg.so" cur "noredist MCG_LIB_PATH=paper_2305_07238_b200/_lib/exp_noredist/libmcg.so" "minb6 MCG_LIB_PATH=paper_2305_07238_b200/_lib/exp_minb6/libmcg.so" cur2 > gpurun_out/r2/ab_c.txt 2>&1
timeout 900 python profiles/scripts/tuning_1080p.py > gpurun_out/r2/tuning_c.json 2> gpurun_out/r2/tuning_c.err
