mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_prims.py -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2u_bench.log 2>&1
python bench.py --no-cpu --steps 10 > gpurun_out/r2u_bench2.log 2>&1
