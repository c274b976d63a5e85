mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
free -g >> gpurun_out/r2a_smi.txt; nproc >> gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/r2a_bench.log 2> gpurun_out/r2a_bench.err; echo bench_rc=$?
