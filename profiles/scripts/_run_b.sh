mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gpu_tests_b.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2/gpu_tests_b.log
timeout 900 python profiles/scripts/fidelity_factors.py --kind italianflat --span 0 --mip 0 > gpurun_out/r2/factors_if.json 2> gpurun_out/r2/factors_if.err
timeout 900 python profiles/scripts/fidelity_factors.py --kind classroom --span 0.999 --mip 0 > gpurun_out/r2/factors_cl.json 2> gpurun_out/r2/factors_cl.err
timeout 900 python profiles/scripts/fidelity_r2.py --ref-runs 1 --gpu-runs 1 --kinds classroom,cornell,bmw --spans 0.999 --mips 3,4 > gpurun_out/r2/fidelity_b.json 2> gpurun_out/r2/fidelity_b.err
