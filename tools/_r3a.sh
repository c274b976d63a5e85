mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py -m gpu -q -x > gpurun_out/r3a_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 20 > gpurun_out/r3a_bench.log 2>&1
HG_RELIN_NR=0 python bench.py --no-cpu --steps 20 > gpurun_out/r3a_bench_nonr.log 2>&1
