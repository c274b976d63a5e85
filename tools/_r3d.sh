mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_encode.py tests/test_gpu_decode.py tests/test_gpu_prims.py -m gpu -q -x > gpurun_out/r3d_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu --steps 20 > gpurun_out/r3d_bench.log 2>&1
ITERS=4 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r3d_e2e.log 2>&1
