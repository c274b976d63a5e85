for s in 0 1; do echo "== dig=$s"; HG_RELIN_DIG=$s timeout 600 python tools/diag_step.py c5 2>&1 | grep "step [45]\|k_relin"; done > gpurun_out/ab18.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t18.log 2>&1; echo t_rc=$?
timeout 600 python tools/prim_sweep.py --ns 8192,16384 --ls 7,15 > gpurun_out/sweep18.log 2>&1
