mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py tests/test_gpu_determinism.py -m gpu -q -x > gpurun_out/r2d_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2d_bench_pipe.log 2>&1; echo bench_rc=$?
HG_RESCALE_PIPE=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2d_bench_nopipe.log 2>&1; echo bench_rc=$?
timeout 600 python tools/diag_step.py c5 > gpurun_out/r2d_diag_c5.log 2>&1; echo diag_rc=$?
