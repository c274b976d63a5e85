mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py tests/test_gpu_dropin.py -m gpu -q -x > gpurun_out/r2g_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2g_bench.log 2>&1; echo bench_rc=$?
HG_RELIN_D32=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2g_bench_nod32.log 2>&1; echo bench_rc=$?
timeout 900 python tools/diag_step.py c4 6 > gpurun_out/r2g_diag_c4.log 2>&1
