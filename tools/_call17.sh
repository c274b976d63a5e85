for s in 0 1; do echo "== dig=$s"; HG_RELIN_DIG=$s timeout 300 python tools/diag_step.py c3 2>&1 | grep "step [45]\|k_relin"; done > gpurun_out/ab17.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t17.log 2>&1; echo t_rc=$?
