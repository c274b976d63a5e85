mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_shard.py tests/test_gpu_determinism.py -m gpu -q -x > gpurun_out/r2v_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2v_bench.log 2>&1
HG_PLANES_FUSION=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2v_bench_nopf.log 2>&1
timeout 600 python tools/diag_step.py c5 6 > gpurun_out/r2v_diag_c5.log 2>&1
