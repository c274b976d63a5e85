timeout 300 python tools/diag_step.py c3 > gpurun_out/diag16.log 2>&1
timeout 300 python tools/e2e_breakdown.py c3 > gpurun_out/e2e16.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t16.log 2>&1; echo t_rc=$?
timeout 600 python tools/prim_sweep.py --ns 8192,16384 --ls 7 > gpurun_out/sweep16.log 2>&1
