mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_determinism.py tests/test_gpu_shard.py tests/test_gpu_dropin.py tests/test_gpu_sampler_plan.py -m gpu -q -x > gpurun_out/r2p_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2p_bench.log 2>&1
HG_PREPAD=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2p_bench_noprepad.log 2>&1
