timeout 900 python -m pytest tests/test_gpu_exec.py tests/test_gpu_io.py tests/test_gpu_sampler_plan.py tests/test_gpu_shard.py -x -q > gpurun_out/t13.log 2>&1; echo t_rc=$?
python bench.py --no-cpu > gpurun_out/bench13.log 2> gpurun_out/bench13.err; echo bench_rc=$?
timeout 300 python tools/e2e_breakdown.py c3 > gpurun_out/e2e13.log 2>&1
