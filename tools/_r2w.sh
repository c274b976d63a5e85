mkdir -p gpurun_out
ITERS=6 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r2w_e2e.log 2>&1
python bench.py --no-cpu --steps 20 > gpurun_out/r2w_bench.log 2>&1
