timeout 300 python tools/diag_step.py c3 2>&1 | grep "step [45]\|k_gemm_tc\|k_split" > gpurun_out/d21.log
timeout 600 python tools/diag_step.py c5 2>&1 | grep "step [45]\|k_gemm_tc\|k_split" >> gpurun_out/d21.log
timeout 900 python -m pytest tests/test_gpu_exec.py tests/test_gpu_prims.py tests/test_gpu_shard.py -x -q > gpurun_out/t21.log 2>&1; echo t_rc=$?
