for s in 0 1; do echo "== overlap=$s"; HG_LANE_OVERLAP=$s timeout 300 python tools/diag_step.py c3 2>&1 | tail -22; done > gpurun_out/ab12.log 2>&1
HG_LANE_OVERLAP=1 timeout 300 python tools/e2e_breakdown.py c3 > gpurun_out/e2e12.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t12.log 2>&1; echo t_rc=$?
