mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exec.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/r2i_pytest.log 2>&1; echo pytest_rc=$?
timeout 900 python tools/diag_step.py c4 8 > gpurun_out/r2i_diag_c4.log 2>&1
python bench.py --config c5 --batch 8192 --no-cpu > gpurun_out/r2i_bench_c5.log 2>&1; echo c5_rc=$?
