for s in 0 1; do echo "== rsplit=$s"; HG_RESCALE_SPLIT13=$s timeout 300 python tools/diag_step.py c3 2>&1 | grep "step [45]\|k_rescale"; done > gpurun_out/ab20.log 2>&1
HG_RESCALE_SPLIT13=1 timeout 900 python -m pytest tests/test_gpu_prims.py tests/test_gpu_exec.py -x -q > gpurun_out/t20.log 2>&1; echo t_rc=$?
