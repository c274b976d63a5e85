mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py tests/test_gpu_dropin.py tests/test_gpu_determinism.py -m gpu -q -x > gpurun_out/r2h_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2h_bench.log 2>&1; echo bench_rc=$?
timeout 900 python tools/diag_step.py c4 8 > gpurun_out/r2h_diag_c4.log 2>&1
