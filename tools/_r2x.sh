mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py tests/test_gpu_sampler.py tests/test_gpu_sampler_plan.py tests/test_gpu_io.py tests/test_gpu_dropin.py -m gpu -q -x > gpurun_out/r2x_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 20 > gpurun_out/r2x_bench.log 2>&1
HG_ENCRYPT_PIPE=0 python bench.py --no-cpu --steps 20 > gpurun_out/r2x_bench_nopipe.log 2>&1
ITERS=4 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r2x_e2e.log 2>&1
