mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_determinism.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/r2n_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2n_bench.log 2>&1
HG_RELIN_RESCALE=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2n_bench_unfused.log 2>&1
timeout 600 python tools/diag_step.py c5 4 > gpurun_out/r2n_diag_c5.log 2>&1
