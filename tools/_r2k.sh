mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py -m gpu -q -x > gpurun_out/r2k_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 10 > gpurun_out/r2k_bench.log 2>&1
timeout 600 python tools/prim_sweep.py --ns 8192,16384 --ls 7 > gpurun_out/r2k_sweep.jsonl 2> gpurun_out/r2k_sweep.err
