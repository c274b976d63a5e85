for s in 0 1; do echo "== l1pf=$s"; HG_RELIN_L1PF=$s timeout 300 python tools/diag_step.py c3 2>&1 | tail -22; done > gpurun_out/ab14.log 2>&1
for s in 0 1; do echo "== l1pf=$s"; HG_LANE_OVERLAP=0 HG_RELIN_L1PF=$s timeout 300 python tools/diag_step.py c3 2>&1 | grep "k_relin_t\|step 5"; done >> gpurun_out/ab14.log 2>&1
timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py -x -q > gpurun_out/t14.log 2>&1; echo t_rc=$?
