mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_dropin.py tests/test_gpu_prims.py -m gpu -q > gpurun_out/r2b_pytest.log 2>&1; echo pytest_rc=$?
free -g; nproc
( time HG_GOLDEN_OUT=gpurun_out timeout 2400 python tests/golden/make_golden.py nets c4 ) > gpurun_out/r2b_c4golden.log 2>&1; echo golden_rc=$?
