mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_gpu_exec.py tests/test_gpu_determinism.py -m gpu -q -x -rs > gpurun_out/r2l_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2l_bench.log 2>&1
