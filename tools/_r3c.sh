mkdir -p gpurun_out
python bench.py --no-cpu --steps 20 > gpurun_out/r3c_bench.log 2>&1
ITERS=4 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r3c_e2e.log 2>&1
timeout 900 python tools/prim_sweep.py --ns 16384 --ls 7 --out gpurun_out/r3c_sweep_14.jsonl > gpurun_out/r3c_sweep_14.log 2>&1
HG_NTT_TWG=1 timeout 900 python tools/prim_sweep.py --ns 16384 --ls 7 --out gpurun_out/r3c_sweep_14_twg.jsonl > gpurun_out/r3c_sweep_14_twg.log 2>&1
timeout 300 python -m pytest tests/test_gpu_prims.py -m gpu -q -x -k "ntt" > gpurun_out/r3c_pytest.log 2>&1
HG_NTT_TWG=1 timeout 300 python -m pytest tests/test_gpu_prims.py -m gpu -q -x -k "ntt" > gpurun_out/r3c_pytest_twg.log 2>&1
