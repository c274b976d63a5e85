mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r3b_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 20 > gpurun_out/r3b_bench.log 2>&1
HG_RELIN_NR=0 python bench.py --no-cpu --steps 20 > gpurun_out/r3b_bench_nonr.log 2>&1
HG_GPU_DECODE=0 python bench.py --no-cpu --steps 20 > gpurun_out/r3b_bench_hostdec.log 2>&1
timeout 600 python tools/e2e_phases.py c3 > gpurun_out/r3b_phases.log 2>&1
ITERS=4 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r3b_e2e.log 2>&1
