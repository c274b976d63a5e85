mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py -m gpu -q -x > gpurun_out/r2j_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2j_bench.log 2>&1
HG_RESCALE_SPLIT13=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2j_bench_nosplit.log 2>&1
HG_TC_MIN_TERMS=16 python bench.py --no-cpu --steps 10 > gpurun_out/r2j_bench_tc16.log 2>&1
HG_TC_MIN_TERMS=16 timeout 600 python tools/diag_step.py c4 4 > gpurun_out/r2j_diag_c4_tc16.log 2>&1
