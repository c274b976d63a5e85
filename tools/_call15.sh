for s in 0 1; do echo "== mix=$s"; HG_RELIN_MIX=$s timeout 300 python tools/diag_step.py c3 2>&1 | grep "step [45]"; done > gpurun_out/ab15.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t15.log 2>&1; echo t_rc=$?
