mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r2c_pytest.log 2>&1; echo pytest_rc=$?
python bench.py --no-cpu-single > gpurun_out/r2c_bench.log 2> gpurun_out/r2c_bench.err; echo bench_rc=$?
