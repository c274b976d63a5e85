mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_exec.py -m gpu -q -x > gpurun_out/r2s_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2s_bench.log 2>&1
HG_LANE_SLOTS=1 python bench.py --no-cpu --steps 10 > gpurun_out/r2s_bench_ls1.log 2>&1
HG_LANE_OVERLAP=0 python bench.py --no-cpu --steps 10 > gpurun_out/r2s_bench_nooverlap.log 2>&1
