mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_prims.py -m gpu -q -x > gpurun_out/r2o_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2o_bench.log 2>&1
HG_RESCALE_STAGE_LIFT=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2o_bench_nostage.log 2>&1
timeout 600 python tools/diag_step.py c5 6 > gpurun_out/r2o_diag_c5.log 2>&1
HG_RELIN_RESCALE=0 timeout 600 python tools/diag_step.py c5 6 > gpurun_out/r2o_diag_c5_unfused.log 2>&1
timeout 900 python tools/diag_step.py c4 5 > gpurun_out/r2o_diag_c4.log 2>&1
