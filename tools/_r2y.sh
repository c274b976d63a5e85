mkdir -p gpurun_out
nproc > gpurun_out/r2y_host.log; free -g >> gpurun_out/r2y_host.log; uptime >> gpurun_out/r2y_host.log
python bench.py --no-cpu --steps 20 > gpurun_out/r2y_bench.log 2>&1
uptime >> gpurun_out/r2y_host.log
timeout 600 python tools/e2e_phases.py c3 > gpurun_out/r2y_phases.log 2>&1
ITERS=6 timeout 600 python tools/e2e_breakdown.py c3 > gpurun_out/r2y_e2e.log 2>&1
python bench.py --no-cpu --steps 20 > gpurun_out/r2y_bench2.log 2>&1
top -b -n 1 | head -20 >> gpurun_out/r2y_host.log
